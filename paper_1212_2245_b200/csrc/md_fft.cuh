// md_fft.cuh -- shared-memory radix-2 FFT building blocks.
//
// Convolution-style pairing: the forward transform is decimation-in-frequency (natural
// order in, bit-reversed order out), the inverse is decimation-in-time (bit-reversed in,
// natural out). Spectra and filters are therefore stored in bit-reversed order and no
// permutation pass is ever executed. Convention matches the reference FourierPlan
// (fft.py:52-117): forward unnormalised, inverse scaled by 1/n by the caller's epilogue.
// Twiddles tw[k] = exp(-2*pi*i*k/n), k < n/2, are tabulated per length at plan time.
#pragma once

#include "md_common.cuh"

namespace md {

// `nl` lines of length n = 2^log2n at s[l * stride + j]; all threads of the block take part.
template <typename C>
__device__ void fft_dif_lines(C *s, int log2n, int nl, int stride, const C *__restrict__ tw) {
    const int n = 1 << log2n;
    const int hb = log2n - 1;                  // log2(n/2)
    const int nb = nl << hb;                   // butterflies per stage
    int tstride = 1;
    for (int lh = hb; lh >= 0; --lh, tstride <<= 1) {
        const int half = 1 << lh;
        for (int b = threadIdx.x; b < nb; b += blockDim.x) {
            const int l = b >> hb;
            const int bb = b & ((n >> 1) - 1);
            const int k = bb & (half - 1);
            const int i0 = ((bb >> lh) << (lh + 1)) + k;
            C *row = s + l * stride;
            C a = row[i0], c = row[i0 + half];
            C w = tw[k * tstride];
            row[i0] = cadd(a, c);
            row[i0 + half] = cmul(csub(a, c), w);
        }
        __syncthreads();
    }
}

// inverse (conjugate twiddles), bit-reversed in -> natural out, unscaled
template <typename C>
__device__ void fft_dit_inv_lines(C *s, int log2n, int nl, int stride, const C *__restrict__ tw) {
    const int n = 1 << log2n;
    const int hb = log2n - 1;
    const int nb = nl << hb;
    int tstride = n >> 1;
    for (int lh = 0; lh <= hb; ++lh, tstride >>= 1) {
        const int half = 1 << lh;
        for (int b = threadIdx.x; b < nb; b += blockDim.x) {
            const int l = b >> hb;
            const int bb = b & ((n >> 1) - 1);
            const int k = bb & (half - 1);
            const int i0 = ((bb >> lh) << (lh + 1)) + k;
            C *row = s + l * stride;
            C t = cmulc(row[i0 + half], tw[k * tstride]);
            C a = row[i0];
            row[i0 + half] = csub(a, t);
            row[i0] = cadd(a, t);
        }
        __syncthreads();
    }
}

}  // namespace md
