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

// Shared-memory position of element j of a line: one pad slot after every 8 elements. The
// radix-4 stages with small spans access elements 8, 32, ... apart; unpadded, 16-byte (f64
// complex) elements at stride 8 all fall into one bank group (16-way conflicts, measured
// 2.8e8 conflicts per two-level pass at 16384^2); padded, they spread over all banks.
// ES = element bytes: 16-byte (complex double) lines pad once per 8 elements, 8-byte (complex
// float) ones once per 16 -- then a half-warp's 8-byte accesses at strides 1, 2, 4, 8, 16 hit
// distinct banks (one pad per 8 left the small-span radix-4 stages 2-4-way conflicted)
template <int ES = 16> __host__ __device__ constexpr int fpad(int j) { return j + (j >> (ES <= 8 ? 4 : 3)); }
// storage length of a padded line of n elements
template <int ES = 16> __host__ __device__ constexpr int fpad_len(int n) { return fpad<ES>(n - 1) + 1; }
// stride between padded lines that are accessed across lines (transposed loads / stores):
// = 1 (mod 8), so 8 consecutive lines fall into 8 different bank groups for 16-byte complex
// elements (and 16 into different bank pairs for 8-byte ones)
template <int ES = 16> __host__ __device__ constexpr int fline_stride(int n) { return ((fpad_len<ES>(n) + 6) & ~7) + 1; }

// `nl` lines of length n = 2^log2n at s[l * stride + fpad(j)]; all threads of the block take part.
// Pairs of radix-2 stages are fused into radix-4 units (4 elements in registers), halving the
// shared-memory round trips and barriers; an odd stage count leaves one radix-2 stage.
template <typename C>
__device__ __forceinline__ C mul_mi(C a) {          // a * (-i)
    C r; r.x = a.y; r.y = -a.x; return r;
}

// Stage-major twiddle table for the STAGED variants: the stage with butterfly half-size h reads
// W_{2h}^k, k < h, at tws[h - 1 + k] (n - 1 entries in all), so consecutive lanes of a stage
// read consecutive entries -- the natural table read at tw[k << shift] strides the banks. Filled
// by a block from the plan's natural table twg[k] = W_n^k, k < n/2.
// BD: the block size when the caller knows it at compile time (0: blockDim.x) -- with the
// length also a compile-time constant the loops below unroll and their index math folds
template <int BD = 0, typename C>
__device__ __forceinline__ void stage_twiddles(C *tws, const C *__restrict__ twg, int log2n) {
    const int n = 1 << log2n;
    const int bd = BD ? BD : (int)blockDim.x;
    for (int i = threadIdx.x; i < n - 1; i += bd) {
        const int lh = 31 - __clz(i + 1), h = 1 << lh;     // stage of entry i
        tws[i] = twg[(i - (h - 1)) << (log2n - 1 - lh)];   // W_{2h}^k = W_n^{k n / 2h}
    }
}

template <bool STAGED = false, int BD = 0, typename C>
__device__ __forceinline__ void fft_dif_lines(C *s, int log2n, int nl, int stride, const C *__restrict__ tw) {
    const int n = 1 << log2n;
    const int bd = BD ? BD : (int)blockDim.x;
    int lh = log2n - 1;
    if (log2n & 1) {                               // lone radix-2 stage, half = n/2
        const int half = n >> 1;
        for (int b = threadIdx.x; b < (nl << lh); b += bd) {
            const int l = b >> lh, k = b & (half - 1);
            C *row = s + l * stride;
            const C a = row[fpad<sizeof(C)>(k)], c = row[fpad<sizeof(C)>(k + half)];
            row[fpad<sizeof(C)>(k)] = cadd(a, c);
            row[fpad<sizeof(C)>(k + half)] = cmul(csub(a, c), tw[STAGED ? half - 1 + k : k]);
        }
        __syncthreads();
        --lh;
    }
    const int lu = log2n - 2;                      // log2(n/4) units per line
    for (; lh >= 1; lh -= 2) {
        const int h = 1 << lh, q = h >> 1;
        for (int u = threadIdx.x; u < (nl << lu); u += bd) {
            const int l = u >> lu, uu = u & ((n >> 2) - 1);
            const int k = uu & (q - 1);
            const int i0 = ((uu >> (lh - 1)) << (lh + 1)) + k;
            C *row = s + l * stride;
            const C x0 = row[fpad<sizeof(C)>(i0)], x1 = row[fpad<sizeof(C)>(i0 + q)], x2 = row[fpad<sizeof(C)>(i0 + h)], x3 = row[fpad<sizeof(C)>(i0 + h + q)];
            const C w1 = STAGED ? tw[h - 1 + k] : tw[k << (log2n - 1 - lh)];      // W_{2h}^k
            const C w2 = STAGED ? tw[q - 1 + k] : tw[k << (log2n - lh)];          // W_h^k
            const C y0 = cadd(x0, x2), y2 = cmul(csub(x0, x2), w1);
            const C y1 = cadd(x1, x3), y3 = cmul(csub(x1, x3), mul_mi(w1));
            row[fpad<sizeof(C)>(i0)] = cadd(y0, y1);
            row[fpad<sizeof(C)>(i0 + q)] = cmul(csub(y0, y1), w2);
            row[fpad<sizeof(C)>(i0 + h)] = cadd(y2, y3);
            row[fpad<sizeof(C)>(i0 + h + q)] = cmul(csub(y2, y3), w2);
        }
        __syncthreads();
    }
}

// inverse (conjugate twiddles), bit-reversed in -> natural out, unscaled
template <bool STAGED = false, int BD = 0, typename C>
__device__ __forceinline__ void fft_dit_inv_lines(C *s, int log2n, int nl, int stride, const C *__restrict__ tw) {
    const int n = 1 << log2n;
    const int bd = BD ? BD : (int)blockDim.x;
    const int hb = log2n - 1;
    const int lu = log2n - 2;
    int lh = 0;
    for (; lh + 1 <= hb; lh += 2) {                // stages half = 2^lh and 2^(lh+1)
        const int q = 1 << lh, h = q << 1;
        for (int u = threadIdx.x; u < (nl << lu); u += bd) {
            const int l = u >> lu, uu = u & ((n >> 2) - 1);
            const int k = uu & (q - 1);
            const int i0 = ((uu >> lh) << (lh + 2)) + k;
            C *row = s + l * stride;
            const C x0 = row[fpad<sizeof(C)>(i0)], x1 = row[fpad<sizeof(C)>(i0 + q)], x2 = row[fpad<sizeof(C)>(i0 + h)], x3 = row[fpad<sizeof(C)>(i0 + h + q)];
            const C w2 = STAGED ? tw[q - 1 + k] : tw[k << (log2n - lh - 1)];      // W_h^k
            const C w1 = STAGED ? tw[h - 1 + k] : tw[k << (log2n - lh - 2)];      // W_{2h}^k
            C t = cmulc(x1, w2);
            const C y0 = cadd(x0, t), y1 = csub(x0, t);
            t = cmulc(x3, w2);
            const C y2 = cadd(x2, t), y3 = csub(x2, t);
            t = cmulc(y2, w1);
            row[fpad<sizeof(C)>(i0)] = cadd(y0, t);
            row[fpad<sizeof(C)>(i0 + h)] = csub(y0, t);
            t = cmulc(y3, mul_mi(w1));
            row[fpad<sizeof(C)>(i0 + q)] = cadd(y1, t);
            row[fpad<sizeof(C)>(i0 + h + q)] = csub(y1, t);
        }
        __syncthreads();
    }
    if (lh == hb) {                                // lone radix-2 stage, half = n/2
        const int half = n >> 1;
        for (int b = threadIdx.x; b < (nl << hb); b += bd) {
            const int l = b >> hb, k = b & (half - 1);
            C *row = s + l * stride;
            const C t = cmulc(row[fpad<sizeof(C)>(k + half)], tw[STAGED ? half - 1 + k : k]);
            const C a = row[fpad<sizeof(C)>(k)];
            row[fpad<sizeof(C)>(k + half)] = csub(a, t);
            row[fpad<sizeof(C)>(k)] = cadd(a, t);
        }
        __syncthreads();
    }
}

}  // namespace md
