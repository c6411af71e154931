// md_fft2d.cu -- 2D FFT passes for the FOURIER_2D scenario with dense kernels (the
// _FourierConvolver2D / wiener_2d path, deconv.py:257-272, 359-376, 660-664; fft.py:165-170,
// 274-280) and for PSF spectra.
//
// A 2D transform is a row pass (length W, contiguous) and a column pass (length H). The
// forward direction is DIF, so a spectrum is held in "storage coordinates" -- bit-reversed
// along both axes -- and filters are computed in the same coordinates; inverse passes are
// DIT and return natural order. Pointwise RRRL work is fused into the row passes:
//   row pass  : [load] -> [inverse DIT] -> epilogue -> [forward DIF of the packed result]
//   col pass  : DIF -> x filter (or conj) -> DIT        (or DIF only, for spectra)
// With this fusion one FOURIER_2D iteration is 4 launches:
//   rows(inv, stage A: b -> W, p; pack p + iW; fwd) -> cols(x conj h) ->
//   rows(inv, stage B: adjoint pair + TV + update; pack u'; fwd) -> cols(x h)
#include "md_fft.cuh"
#include "md_plane.h"

namespace md {

// TV divergence at (y, x) straight from global memory (the row pass owns one row only)
template <typename T>
__device__ T tv_div_global(const T *__restrict__ u, int H, int W, int y, int x, T eps_r2) {
    auto at = [&](int yy, int xx) { return __ldg(u + (int64_t)yy * W + xx); };
    auto gfun = [&](int yy, int xx) {
        const T c = at(yy, xx);
        T q = T(0);
        if (xx + 1 < W) { const T d = at(yy, xx + 1) - c; q += d * d; }
        if (xx > 0) { const T d = c - at(yy, xx - 1); q += d * d; }
        if (yy + 1 < H) { const T d = at(yy + 1, xx) - c; q += d * d; }
        if (yy > 0) { const T d = c - at(yy - 1, xx); q += d * d; }
        return T(0.5) / sqrt(T(0.5) * q + eps_r2);
    };
    const T u0 = at(y, x), gc = gfun(y, x);
    T d = T(0);
    if (x + 1 < W) d += (gc + gfun(y, x + 1)) * (at(y, x + 1) - u0);
    if (x > 0) d -= (gfun(y, x - 1) + gc) * (u0 - at(y, x - 1));
    if (y + 1 < H) d += (gc + gfun(y + 1, x)) * (at(y + 1, x) - u0);
    if (y > 0) d -= (gfun(y - 1, x) + gc) * (u0 - at(y - 1, x));
    return d;
}

template <typename T>
__global__ void __launch_bounds__(256)
k_fft2_rows(Fft2Args a, int rb) {
    // `rb` consecutive rows per block (all threads busy in every FFT stage)
    using C = cx_t<T>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *s = reinterpret_cast<C *>(smem_raw);
    const int H = a.H, W = a.W, lw = a.log2W;
    const int y0 = blockIdx.x * rb;
    const int64_t fsz = (int64_t)H * W;
    const int64_t fr = blockIdx.y;
    const int64_t base = fr * fsz + (int64_t)y0 * W;      // rb rows are contiguous
    const int ne = rb * W;
    C *z = static_cast<C *>(a.z);
    const C *tw = static_cast<const C *>(a.twW);

    if (a.load == R_LOAD_COMPLEX) {
        for (int i = threadIdx.x; i < ne; i += blockDim.x) s[i] = z[base + i];
    } else {
        const T *ra = static_cast<const T *>(a.ra);
        const T *rb_ = static_cast<const T *>(a.rb);
        for (int i = threadIdx.x; i < ne; i += blockDim.x) s[i] = mkc<T>(ra[base + i], rb_ ? rb_[base + i] : T(0));
    }
    __syncthreads();
    if (a.inv && lw > 0) fft_dit_inv_lines(s, lw, rb, W, tw);

    const T scale = T(a.scale), floor = T(a.floor);
    if (a.epi != R_EPI_NONE) {
        for (int i = threadIdx.x; i < ne; i += blockDim.x) {
            const C v = s[i];
            const int64_t o = base + i;
            C packed = mkc<T>(T(0), T(0));
            if (a.epi == R_EPI_STORE_PAIR) {
                static_cast<T *>(a.oa)[o] = v.x * scale;
                if (a.ob) static_cast<T *>(a.ob)[o] = v.y * scale;
            } else if (a.epi == R_EPI_WIENER) {
                T w = v.x * scale;
                if (floor > T(0)) w = w > floor ? w : floor;     // u0 = max(Wiener, floor)
                static_cast<T *>(a.oa)[o] = w;
                if (a.ob) {
                    const T fv = static_cast<const T *>(a.f)[o];
                    static_cast<T *>(a.ob)[o] = fv > floor ? fv : floor;
                }
                packed = mkc<T>(w, T(0));
            } else if (a.epi == R_EPI_STAGE_A) {
                T b = v.x * scale;
                b = b > T(kGuard) ? b : T(kGuard);
                const T fp = static_cast<const T *>(a.f)[o];
                const T ratio = fp / b;
                if (a.robust) {
                    const T wv = robust_weight_floored<T>(a.lut, fp, b, T(a.eps_d2));
                    packed = mkc<T>(wv * ratio, wv);
                } else {
                    packed = mkc<T>(ratio, T(0));
                }
            } else {  // R_EPI_STAGE_B
                const T *u = static_cast<const T *>(a.u) + fr * fsz;
                const int y = y0 + (i >> lw), x = i & (W - 1);
                const T uv = u[(int64_t)y * W + x];
                const T d = a.has_d ? tv_div_global<T>(u, H, W, y, x, T(a.eps_r2)) : T(0);
                const T un = a.robust ? combine_px<T, true>(uv, v.x * scale, v.y * scale, d, T(a.alpha), a.has_d != 0)
                                      : combine_px<T, false>(uv, v.x * scale, T(0), d, T(a.alpha), a.has_d != 0);
                static_cast<T *>(a.oa)[o] = un;
                packed = mkc<T>(un, T(0));
            }
            s[i] = packed;
        }
        __syncthreads();
    }
    if (a.fwd_after) {
        if (lw > 0) fft_dif_lines(s, lw, rb, W, tw);
        for (int i = threadIdx.x; i < ne; i += blockDim.x) z[base + i] = s[i];
    } else if (a.epi == R_EPI_NONE) {
        for (int i = threadIdx.x; i < ne; i += blockDim.x) z[base + i] = s[i];
    }
}

template <typename T>
__global__ void __launch_bounds__(256)
k_fft2_cols(Fft2Args a, int cw) {
    using C = cx_t<T>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *s = reinterpret_cast<C *>(smem_raw);
    const int H = a.H, W = a.W, cs = H + 1;
    const int x0 = blockIdx.x * cw;
    const int64_t base = blockIdx.y * (int64_t)H * W;
    C *z = static_cast<C *>(a.z);
    const C *tw = static_cast<const C *>(a.twH);
    for (int idx = threadIdx.x; idx < cw * H; idx += blockDim.x) {
        const int y = idx / cw, c = idx - y * cw;
        if (x0 + c < W) s[c * cs + y] = z[base + (int64_t)y * W + x0 + c];
        else s[c * cs + y] = mkc<T>(T(0), T(0));
    }
    __syncthreads();
    if (a.log2H > 0) fft_dif_lines(s, a.log2H, cw, cs, tw);
    if (a.filt) {
        const C *filt = static_cast<const C *>(a.filt);
        for (int idx = threadIdx.x; idx < cw * H; idx += blockDim.x) {
            const int c = idx / H, y = idx - c * H;
            if (x0 + c >= W) continue;
            const C f = __ldg(filt + (int64_t)y * W + x0 + c);
            s[c * cs + y] = a.conj_filt ? cmulc(s[c * cs + y], f) : cmul(s[c * cs + y], f);
        }
        __syncthreads();
    }
    if (a.col_inv && a.log2H > 0) fft_dit_inv_lines(s, a.log2H, cw, cs, tw);
    for (int idx = threadIdx.x; idx < cw * H; idx += blockDim.x) {
        const int y = idx / cw, c = idx - y * cw;
        if (x0 + c < W) z[base + (int64_t)y * W + x0 + c] = s[c * cs + y];
    }
}

template <typename T>
cudaError_t launch_fft2_rows(const Fft2Args &a, int64_t batch, cudaStream_t st) {
    int rb = 2048 / a.W;                      // ~2048 elements per block
    rb = rb < 1 ? 1 : (rb > a.H ? a.H : rb);
    const size_t smem = (size_t)rb * a.W * sizeof(cx_t<T>);
    cudaError_t e = cudaFuncSetAttribute(k_fft2_rows<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t fr = (int64_t)a.H * a.W;
    for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
        const int nb = (int)((batch - b0) < 65535 ? (batch - b0) : 65535);
        Fft2Args ab = a;
        auto sh = [&](const void *p, size_t es) -> const void * {
            return p ? static_cast<const char *>(p) + b0 * fr * es : nullptr;
        };
        ab.ra = sh(a.ra, sizeof(T));
        ab.rb = sh(a.rb, sizeof(T));
        ab.z = const_cast<void *>(sh(a.z, sizeof(cx_t<T>)));
        ab.oa = const_cast<void *>(sh(a.oa, sizeof(T)));
        ab.ob = const_cast<void *>(sh(a.ob, sizeof(T)));
        ab.f = sh(a.f, sizeof(T));
        ab.u = sh(a.u, sizeof(T));
        k_fft2_rows<T><<<dim3(a.H / rb, nb), 256, smem, st>>>(ab, rb);
    }
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_fft2_cols(const Fft2Args &a, int64_t batch, cudaStream_t st) {
    int cw = 4096 / a.H;
    cw = cw > 16 ? 16 : (cw < 1 ? 1 : cw);
    const size_t smem = (size_t)cw * (a.H + 1) * sizeof(cx_t<T>);
    cudaError_t e = cudaFuncSetAttribute(k_fft2_cols<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t fr = (int64_t)a.H * a.W;
    for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
        const int nb = (int)((batch - b0) < 65535 ? (batch - b0) : 65535);
        Fft2Args ab = a;
        ab.z = static_cast<char *>(a.z) + b0 * fr * sizeof(cx_t<T>);
        k_fft2_cols<T><<<dim3((a.W + cw - 1) / cw, nb), 256, smem, st>>>(ab, cw);
    }
    return cudaGetLastError();
}

template cudaError_t launch_fft2_rows<double>(const Fft2Args &, int64_t, cudaStream_t);
template cudaError_t launch_fft2_rows<float>(const Fft2Args &, int64_t, cudaStream_t);
template cudaError_t launch_fft2_cols<double>(const Fft2Args &, int64_t, cudaStream_t);
template cudaError_t launch_fft2_cols<float>(const Fft2Args &, int64_t, cudaStream_t);

}  // namespace md
