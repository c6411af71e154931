// md_fft_api.cu -- natural-order complex FFTs of contiguous lines: the device side of the
// reference's public transform API (FourierPlan.forward / inverse, fft.py:52-117, and what is
// built on it: fft_forward_real / fft_inverse_real, fft2_forward / fft2_inverse,
// apply_column_filter, filter_real_pair, fft.py:144-280).
//
// The pipeline kernels never permute (spectra stay in bit-reversed or two-level storage order,
// matched by their filters); a public transform must return natural order. Lengths that fit one
// block (n <= 4096 complex128 / 8192 complex64) run in shared memory: the forward transform is
// the DIF network with its bit-reversed output gathered back to natural order on the store, the
// inverse places its natural-order input at bit-reversed positions and runs the DIT network.
// Longer lines (up to 65536) run the two-level passes of md_fft_big.cu and a permutation
// between natural and their storage order (position q + N1 p holds k = rev_N2(p) + N2 rev_N1(q)).
// Convention as the reference: forward unnormalised, inverse scaled by 1/n.
#include "md_fft.cuh"
#include "md_fft_big.h"

namespace md {

__device__ __forceinline__ int brev_bits(int x, int bits) {
    return bits == 0 ? 0 : (int)(__brev((unsigned)x) >> (32 - bits));
}

// G lines of n = 2^log2n per block, in place
template <typename T>
__global__ void __launch_bounds__(256) k_fft_lines_nat(cx_t<T> *z, int log2n, int64_t lines, int G,
                                                       const cx_t<T> *__restrict__ twg, int inverse) {
    using C = cx_t<T>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *s = reinterpret_cast<C *>(smem_raw);
    const int n = 1 << log2n, ls = fline_stride<sizeof(C)>(n);
    C *tw = s + G * ls;
    stage_twiddles(tw, twg, log2n);
    const int64_t l0 = (int64_t)blockIdx.x * G;
    const int gl = (int)(lines - l0 < G ? lines - l0 : G);
    C *zb = z + l0 * n;
    for (int i = threadIdx.x; i < gl * n; i += blockDim.x) {
        const int g = i >> log2n, j = i & (n - 1);
        const C v = zb[i];
        s[g * ls + fpad<sizeof(C)>(inverse ? brev_bits(j, log2n) : j)] = v;
    }
    for (int i = gl * n + threadIdx.x; i < G * n; i += blockDim.x) {   // idle lines of a ragged block
        const int g = i >> log2n, j = i & (n - 1);
        s[g * ls + fpad<sizeof(C)>(j)] = mkc<T>(T(0), T(0));
    }
    __syncthreads();
    if (log2n > 0) {
        if (inverse) fft_dit_inv_lines<true>(s, log2n, G, ls, tw);
        else fft_dif_lines<true>(s, log2n, G, ls, tw);
    }
    const T scale = inverse ? T(1) / T(n) : T(1);
    for (int i = threadIdx.x; i < gl * n; i += blockDim.x) {
        const int g = i >> log2n, k = i & (n - 1);
        const C v = s[g * ls + fpad<sizeof(C)>(inverse ? k : brev_bits(k, log2n))];
        zb[i] = inverse ? cscale(v, scale) : v;
    }
}

// natural <-> two-level storage order of lines of N = N1 * N2 (to_natural: out[k] = in[pos(k)])
template <typename T>
__global__ void k_fft_perm(const cx_t<T> *__restrict__ in, cx_t<T> *__restrict__ out, int l1, int l2,
                           int64_t total, int to_natural) {
    const int N1 = 1 << l1, N2 = 1 << l2, N = N1 * N2;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t line = i / N;
        const int r = (int)(i - line * N);
        if (to_natural) {                       // r = natural k -> storage position
            const int p = brev_bits(r & (N2 - 1), l2), q = brev_bits(r >> l2, l1);
            out[i] = in[line * N + q + N1 * p];
        } else {                                // r = storage position q + N1 p -> natural k
            const int q = r & (N1 - 1), p = r >> l1;
            out[i] = in[line * N + brev_bits(p, l2) + N2 * brev_bits(q, l1)];
        }
    }
}

template <typename T>
int fft_lines_max_single() { return sizeof(T) == 8 ? 4096 : 8192; }

template <typename T>
cudaError_t launch_fft_lines_nat(void *z, int n, int64_t lines, const void *tw, int inverse, cudaStream_t st) {
    using C = cx_t<T>;
    int log2n = 0;
    while ((1 << log2n) < n) ++log2n;
    const int G = std::max(1, std::min(16, 2048 / n));
    const size_t smem = ((size_t)G * fline_stride<sizeof(C)>(n) + n + 1) * sizeof(C);
    cudaError_t e = func_smem_attr((const void *)k_fft_lines_nat<T>, smem);
    if (e != cudaSuccess) return e;
    const int64_t blocks = (lines + G - 1) / G;
    if (blocks > 0x7fffffff) return cudaErrorInvalidValue;
    k_fft_lines_nat<T><<<(unsigned)blocks, 256, smem, st>>>(static_cast<C *>(z), log2n, lines, G,
                                                          static_cast<const C *>(tw), inverse);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_fft_perm(const void *in, void *out, const BigAxis &ax, int64_t lines, int to_natural,
                            cudaStream_t st) {
    const int64_t total = lines * (int64_t)ax.N;
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 64);
    k_fft_perm<T><<<blocks, 256, 0, st>>>(static_cast<const cx_t<T> *>(in), static_cast<cx_t<T> *>(out), ax.l1,
                                         ax.l2, total, to_natural);
    return cudaGetLastError();
}

template cudaError_t launch_fft_lines_nat<double>(void *, int, int64_t, const void *, int, cudaStream_t);
template cudaError_t launch_fft_lines_nat<float>(void *, int, int64_t, const void *, int, cudaStream_t);
template cudaError_t launch_fft_perm<double>(const void *, void *, const BigAxis &, int64_t, int, cudaStream_t);
template cudaError_t launch_fft_perm<float>(const void *, void *, const BigAxis &, int64_t, int, cudaStream_t);
template int fft_lines_max_single<double>();
template int fft_lines_max_single<float>();

}  // namespace md
