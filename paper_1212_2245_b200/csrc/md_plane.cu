// md_plane.cu -- kernels for 2D PSFs with direct (sparse-tap) convolution, periodic
// (FOURIER_2D semantics, deconv.py:359-376, equal to the FFT convolver up to rounding) or
// clamped (_SpatialConvolver / convolve_array, deconv.py:295-307, conv.py:85-116); plus the
// TV divergence and the step-level elementwise kernels of the convolver-protocol API.
//
// One RRRL iteration = two launches (the adjoint needs p and W at PSF-extent distance):
//   k_stage_a_plane : b = max(h*u, guard); W = phi'(r_f(b)); p = W f / b    (deconv.py:415-418, 142-162)
//   k_stage_b_plane : num, den = h~ * (p, W); D = div(psi' grad u); u' = u num / den
//                     (deconv.py:421-446, 187-213)
#include "md_internal.h"
#include "md_plane.h"

namespace md {

constexpr int PT = 32;          // output tile edge
constexpr int PTHREADS = 256;   // 32 x 8

__device__ __forceinline__ int resolve2(int k, int n, int periodic) {
    // a tile plus halo may be larger than a small frame: a full wrap (see pf_resolve)
    if (periodic) {
        k = k < 0 ? k + n : (k >= n ? k - n : k);
        if ((unsigned)k >= (unsigned)n) {
            k %= n;
            k = k < 0 ? k + n : k;
        }
        return k;
    }
    return k < 0 ? 0 : (k >= n ? n - 1 : k);
}

// load rows [y0-ht, y0+PT+hb) x cols [x0-hl, x0+PT+hr) of a frame, boundary-resolved
template <typename T>
__device__ void load_tile(T *s, int ss, const T *__restrict__ src, int H, int W, int y0, int x0,
                          int ht, int hb, int hl, int hr, int periodic) {
    const int rows = PT + ht + hb, cols = PT + hl + hr;
    for (int idx = threadIdx.x; idx < rows * cols; idx += blockDim.x) {
        const int i = idx / cols, j = idx - i * cols;
        const int y = resolve2(y0 - ht + i, H, periodic);
        const int x = resolve2(x0 - hl + j, W, periodic);
        s[i * ss + j] = src[(int64_t)y * W + x];
    }
}

// u tile with a 2-pixel halo (rows y0-2.., cols x0-2..), zero outside the image
template <typename T>
__device__ void load_tile_halo2(T *s, int ss, const T *__restrict__ src, int H, int W, int y0, int x0) {
    const int rows = PT + 4, cols = PT + 4;
    for (int idx = threadIdx.x; idx < rows * cols; idx += blockDim.x) {
        const int i = idx / cols, j = idx - i * cols;
        const int y = y0 - 2 + i, x = x0 - 2 + j;
        s[i * ss + j] = (y >= 0 && y < H && x >= 0 && x < W) ? src[(int64_t)y * W + x] : T(0);
    }
}

// diffusivity g on rows y0-1..y0+PT, cols x0-1..x0+PT (deconv.py:191-203)
template <typename T>
__device__ void tv_g_tile(const T *su, int sus, T *sg, int sgs, int H, int W, int y0, int x0, T eps_r2) {
    const int rows = PT + 2, cols = PT + 2;
    for (int idx = threadIdx.x; idx < rows * cols; idx += blockDim.x) {
        const int i = idx / cols, j = idx - i * cols;
        const int y = y0 - 1 + i, x = x0 - 1 + j;
        if (y < 0 || y >= H || x < 0 || x >= W) continue;
        const T *r = su + (i + 1) * sus + (j + 1);
        const T c = r[0];
        T q = T(0);
        if (x + 1 < W) { const T d = r[1] - c; q += d * d; }
        if (x > 0) { const T d = c - r[-1]; q += d * d; }
        if (y + 1 < H) { const T d = r[sus] - c; q += d * d; }
        if (y > 0) { const T d = c - r[-sus]; q += d * d; }
        sg[i * sgs + j] = T(0.5) / sqrt(T(0.5) * q + eps_r2);
    }
}

// divergence D at tile position (ty, tx) (global (y, x)); x fluxes first (deconv.py:204-213)
template <typename T>
__device__ __forceinline__ T tv_div_at(const T *su, int sus, const T *sg, int sgs, int ty, int tx,
                                       int y, int x, int H, int W) {
    const T *r = su + (ty + 2) * sus + (tx + 2);
    const T *g = sg + (ty + 1) * sgs + (tx + 1);
    const T u = r[0], gc = g[0];
    T d = T(0);
    if (x + 1 < W) d += (gc + g[1]) * (r[1] - u);
    if (x > 0) d -= (g[-1] + gc) * (u - r[-1]);
    if (y + 1 < H) d += (gc + g[sgs]) * (r[sus] - u);
    if (y > 0) d -= (g[-sgs] + gc) * (u - r[-sus]);
    return d;
}

template <typename T>
__device__ __forceinline__ T tap_sum(const T *s, int ss, int ty, int tx, const PlaneTap *taps, int nt,
                                     int oy, int ox) {
    T acc = T(0);
    const T *base = s + (ty + oy) * ss + (tx + ox);
    for (int t = 0; t < nt; ++t) acc += T(taps[t].w) * base[taps[t].dy * ss + taps[t].dx];
    return acc;
}

// the same sum with the reference's rounding (conv.py:85-116: acc += w * shifted, a multiply
// and an add per tap, in tap order) -- the public convolve / synth_blur path, which must
// reproduce the reference's quantised test inputs bit for bit at any size; float keeps FMAs
__device__ __forceinline__ double tap_sum_ref(const double *s, int ss, int ty, int tx, const PlaneTap *taps, int nt,
                                              int oy, int ox) {
    double acc = 0.0;
    const double *base = s + (ty + oy) * ss + (tx + ox);
    for (int t = 0; t < nt; ++t) acc = __dadd_rn(acc, __dmul_rn(taps[t].w, base[taps[t].dy * ss + taps[t].dx]));
    return acc;
}
__device__ __forceinline__ float tap_sum_ref(const float *s, int ss, int ty, int tx, const PlaneTap *taps, int nt,
                                             int oy, int ox) {
    return tap_sum<float>(s, ss, ty, tx, taps, nt, oy, ox);
}

template <typename T, bool ROBUST>
__global__ void __launch_bounds__(PTHREADS)
k_stage_a_plane(StagePlaneArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    PlaneTap *st = reinterpret_cast<PlaneTap *>(smem_raw);
    T *su = reinterpret_cast<T *>(st + a.blur.nt);
    const int H = a.H, W = a.W;
    const int64_t fsz = (int64_t)H * W;
    const int64_t fr = blockIdx.z;
    const T *u = static_cast<const T *>(a.u) + fr * fsz;
    const T *f = static_cast<const T *>(a.f) + fr * fsz;
    T *p = static_cast<T *>(a.p) + fr * fsz;
    T *w = ROBUST ? static_cast<T *>(a.w) + fr * fsz : nullptr;
    const int y0 = blockIdx.y * PT, x0 = blockIdx.x * PT;
    const PlaneHalo &h = a.blur;
    const int ss = PT + h.hl + h.hr + 1;
    for (int t = threadIdx.x; t < h.nt; t += blockDim.x) st[t] = a.blur_taps[t];
    load_tile<T>(su, ss, u, H, W, y0, x0, h.ht, h.hb, h.hl, h.hr, a.periodic);
    __syncthreads();
    const T eps_d2 = T(a.eps_d2), floor = T(a.floor);
    for (int k = threadIdx.x; k < PT * PT; k += blockDim.x) {
        const int ty = k / PT, tx = k - ty * PT;
        const int y = y0 + ty, x = x0 + tx;
        if (y >= H || x >= W) continue;
        T b = tap_sum<T>(su, ss, ty, tx, st, h.nt, h.ht, h.hl);
        b = b > T(kGuard) ? b : T(kGuard);
        const int64_t o = (int64_t)y * W + x;
        T fv = f[o];
        if (a.floor_f) fv = fv > floor ? fv : floor;
        const T ratio = fv / b;
        if (ROBUST) {
            const T wv = a.general_weight ? robust_weight_general<T>(a.lut, fv, b, eps_d2, floor)
                                          : robust_weight_floored<T>(a.lut, fv, b, eps_d2);
            w[o] = wv;
            p[o] = wv * ratio;
        } else {
            p[o] = ratio;
        }
    }
}

template <typename T, bool ROBUST>
__global__ void __launch_bounds__(PTHREADS)
k_stage_b_plane(StagePlaneArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    PlaneTap *st = reinterpret_cast<PlaneTap *>(smem_raw);
    const PlaneHalo &h = a.adj;
    const int ss = PT + h.hl + h.hr + 1;
    const int srows = PT + h.ht + h.hb;
    T *sp = reinterpret_cast<T *>(st + h.nt);
    T *sw = sp + srows * ss;
    T *su = ROBUST ? sw + srows * ss : sw;
    const int sus = PT + 5;
    T *sg = su + (PT + 4) * sus;
    const int sgs = PT + 3;
    const int H = a.H, W = a.W;
    const int64_t fsz = (int64_t)H * W;
    const int64_t fr = blockIdx.z;
    const T *u = static_cast<const T *>(a.u) + fr * fsz;
    const T *p = static_cast<const T *>(a.p) + fr * fsz;
    const T *w = ROBUST ? static_cast<const T *>(a.w) + fr * fsz : nullptr;
    T *uo = static_cast<T *>(a.u_out) + fr * fsz;
    const int y0 = blockIdx.y * PT, x0 = blockIdx.x * PT;
    for (int t = threadIdx.x; t < h.nt; t += blockDim.x) st[t] = a.adj_taps[t];
    load_tile<T>(sp, ss, p, H, W, y0, x0, h.ht, h.hb, h.hl, h.hr, a.periodic);
    if (ROBUST) load_tile<T>(sw, ss, w, H, W, y0, x0, h.ht, h.hb, h.hl, h.hr, a.periodic);
    load_tile_halo2<T>(su, sus, u, H, W, y0, x0);
    __syncthreads();
    if (a.has_d) {
        tv_g_tile<T>(su, sus, sg, sgs, H, W, y0, x0, T(a.eps_r2));
        __syncthreads();
    }
    const T alpha = T(a.alpha);
    for (int k = threadIdx.x; k < PT * PT; k += blockDim.x) {
        const int ty = k / PT, tx = k - ty * PT;
        const int y = y0 + ty, x = x0 + tx;
        if (y >= H || x >= W) continue;
        const T num = tap_sum<T>(sp, ss, ty, tx, st, h.nt, h.ht, h.hl);
        const T den = ROBUST ? tap_sum<T>(sw, ss, ty, tx, st, h.nt, h.ht, h.hl) : T(0);
        const T d = a.has_d ? tv_div_at<T>(su, sus, sg, sgs, ty, tx, y, x, H, W) : T(0);
        const T uv = su[(ty + 2) * sus + tx + 2];
        uo[(int64_t)y * W + x] = combine_px<T, ROBUST>(uv, num, den, d, alpha, a.has_d != 0);
    }
}

// plain convolution of a (pair of) frame(s) with a tap list (convolver.blur / adjoint / adjoint_pair)
template <typename T>
__global__ void __launch_bounds__(PTHREADS)
k_conv_plane(ConvPlaneArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    PlaneTap *st = reinterpret_cast<PlaneTap *>(smem_raw);
    const PlaneHalo &h = a.h;
    const int ss = PT + h.hl + h.hr + 1;
    T *s = reinterpret_cast<T *>(st + h.nt);
    const int H = a.H, W = a.W;
    const int64_t fsz = (int64_t)H * W;
    const T *in = static_cast<const T *>(a.in) + blockIdx.z * fsz;
    T *out = static_cast<T *>(a.out) + blockIdx.z * fsz;
    const int y0 = blockIdx.y * PT, x0 = blockIdx.x * PT;
    for (int t = threadIdx.x; t < h.nt; t += blockDim.x) st[t] = a.taps[t];
    load_tile<T>(s, ss, in, H, W, y0, x0, h.ht, h.hb, h.hl, h.hr, a.periodic);
    __syncthreads();
    for (int k = threadIdx.x; k < PT * PT; k += blockDim.x) {
        const int ty = k / PT, tx = k - ty * PT;
        const int y = y0 + ty, x = x0 + tx;
        if (y >= H || x >= W) continue;
        out[(int64_t)y * W + x] = tap_sum_ref(s, ss, ty, tx, st, h.nt, h.ht, h.hl);
    }
}

// D = div(psi'(|grad u|^2) grad u) (diffusion_term, deconv.py:216-228)
template <typename T>
__global__ void __launch_bounds__(PTHREADS)
k_diffusion(const T *__restrict__ u, T *__restrict__ out, int H, int W, T eps_r2) {
    __shared__ T su[(PT + 4) * (PT + 5)];
    __shared__ T sg[(PT + 2) * (PT + 3)];
    const int64_t fsz = (int64_t)H * W;
    u += blockIdx.z * fsz;
    out += blockIdx.z * fsz;
    const int y0 = blockIdx.y * PT, x0 = blockIdx.x * PT;
    load_tile_halo2<T>(su, PT + 5, u, H, W, y0, x0);
    __syncthreads();
    tv_g_tile<T>(su, PT + 5, sg, PT + 3, H, W, y0, x0, eps_r2);
    __syncthreads();
    for (int k = threadIdx.x; k < PT * PT; k += blockDim.x) {
        const int ty = k / PT, tx = k - ty * PT;
        const int y = y0 + ty, x = x0 + tx;
        if (y >= H || x >= W) continue;
        out[(int64_t)y * W + x] = tv_div_at<T>(su, PT + 5, sg, PT + 3, ty, tx, y, x, H, W);
    }
}

// robust weight, general (small-observation) or floored form (robust_weight, deconv.py:165-180)
template <typename T>
__global__ void k_robust_weight(const T *__restrict__ f, const T *__restrict__ b, T *__restrict__ out,
                                int64_t n, T eps2, T floor, int floored, LutView lut) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = floored ? robust_weight_floored<T>(lut, f[i], b[i], eps2)
                         : robust_weight_general<T>(lut, f[i], b[i], eps2, floor);
}

// r1 through the device divergence table (DivergenceLut.r1, deconv.py:114-134)
template <typename T>
__global__ void k_lut_r1(const T *__restrict__ x, T *__restrict__ out, int64_t n, LutView lut) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = r1_lut<T>(lut, x[i]);
}

// DivergenceLut.r1 as the public API evaluates it (deconv.py:114-134), in the reference's
// rounding order: (T[i+1] - T[i]) * t + T[i] and slope * x + intercept as separate roundings
// (NumPy applies them as separate array operations; the in-kernel form contracts to FMAs)
__global__ void k_lut_r1_ref(const double *__restrict__ x, double *__restrict__ out, int64_t n, LutView lut) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double xi = x[i];
        double pos = __dmul_rn(__dsub_rn(xi < kLutUpper ? xi : kLutUpper, kLutDelta), kLutInvStep);
        long long idx = (long long)pos;                   // astype(int64): truncation toward zero
        idx = idx < 0 ? 0 : (idx > kLutCount - 2 ? kLutCount - 2 : idx);
        pos = __dsub_rn(pos, (double)idx);
        const double lo = lut.t64[idx], hi = lut.t64[idx + 1];
        double r = __dadd_rn(__dmul_rn(__dsub_rn(hi, lo), pos), lo);
        if (xi > kLutUpper) r = __dadd_rn(__dmul_rn(kLutSlope, xi), kLutIntercept);
        if (xi < kLutDirectBelow) r = __dsub_rn(__dsub_rn(xi, 1.0), log(xi));
        out[i] = r;
    }
}

// ratio = f / b, optionally times w (first half of _combine)
template <typename T>
__global__ void k_ratio(const T *__restrict__ f, const T *__restrict__ b, const T *__restrict__ w,
                        T *__restrict__ out, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const T r = f[i] / b[i];
        out[i] = w ? w[i] * r : r;
    }
}

// second half of _combine given num (and den when a weight is present)
template <typename T>
__global__ void k_combine(const T *__restrict__ u, const T *__restrict__ num, const T *__restrict__ den,
                          const T *__restrict__ d, T *__restrict__ out, int64_t n, T alpha) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const bool has_d = d != nullptr && alpha != T(0);
        const T dv = has_d ? d[i] : T(0);
        out[i] = den ? combine_px<T, true>(u[i], num[i], den[i], dv, alpha, has_d)
                     : combine_px<T, false>(u[i], num[i], T(0), dv, alpha, has_d);
    }
}

template <typename T>
__global__ void k_guard(T *__restrict__ x, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = x[i] > T(kGuard) ? x[i] : T(kGuard);
}

template <typename T>
__global__ void k_min_partial(const T *__restrict__ x, int64_t n, double *__restrict__ partial) {
    __shared__ double red[256];
    double v = 1e308;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double t = (double)x[i];
        v = t < v ? t : v;
    }
    red[threadIdx.x] = v;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s && red[threadIdx.x + s] < red[threadIdx.x]) red[threadIdx.x] = red[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

template <typename T>
__global__ void k_convert(const void *__restrict__ in, void *__restrict__ out, int64_t n, int to_double) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (to_double) static_cast<double *>(out)[i] = (double)static_cast<const T *>(in)[i];
        else static_cast<T *>(out)[i] = (T) static_cast<const double *>(in)[i];
    }
}

template <typename T>
__global__ void k_convert_in(const void *__restrict__ in, int in_type, T *__restrict__ out, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        T v;
        if (in_type == 2) v = T(static_cast<const unsigned char *>(in)[i]);
        else if (in_type == 1) v = T(static_cast<const float *>(in)[i]);
        else v = T(static_cast<const double *>(in)[i]);
        out[i] = v;
    }
}

template <typename T>
__global__ void k_convert_out(const T *__restrict__ in, void *__restrict__ out, int out_type, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (out_type == 1) {
            static_cast<float *>(out)[i] = (float)in[i];
        } else if (out_type == 2) {
            // 8-bit grey, the reference's write_pgm rule: clip(floor(v + 0.5), 0, 255) (pgm.py:56-58)
            T v = floor(in[i] + T(0.5));
            v = v < T(0) ? T(0) : (v > T(255) ? T(255) : v);
            static_cast<unsigned char *>(out)[i] = (unsigned char)v;
        } else {
            static_cast<double *>(out)[i] = (double)in[i];
        }
    }
}

// --------------------------------------------------------------------------------------
// launchers

static inline int ew_blocks(int64_t n) {
    int64_t b = (n + 255) / 256;
    return (int)(b > 148 * 32 ? 148 * 32 : (b < 1 ? 1 : b));
}

template <typename T>
size_t stage_b_smem(const PlaneHalo &h, bool robust) {
    const size_t tile = (size_t)(PT + h.ht + h.hb) * (PT + h.hl + h.hr + 1);
    return h.nt * sizeof(PlaneTap) + ((robust ? 2 : 1) * tile + (PT + 4) * (PT + 5) + (PT + 2) * (PT + 3)) * sizeof(T);
}

template <typename T>
cudaError_t launch_stage_plane(const StagePlaneArgs &a, bool robust, int64_t batch, cudaStream_t st) {
    const dim3 grid0((a.W + PT - 1) / PT, (a.H + PT - 1) / PT, 1);
    const size_t sa = a.blur.nt * sizeof(PlaneTap) +
                      (size_t)(PT + a.blur.ht + a.blur.hb) * (PT + a.blur.hl + a.blur.hr + 1) * sizeof(T);
    const size_t sb = stage_b_smem<T>(a.adj, robust);
    auto ka = robust ? k_stage_a_plane<T, true> : k_stage_a_plane<T, false>;
    auto kb = robust ? k_stage_b_plane<T, true> : k_stage_b_plane<T, false>;
    cudaError_t e = func_smem_attr((const void *)ka, sa);
    if (e == cudaSuccess) e = func_smem_attr((const void *)kb, sb);
    if (e != cudaSuccess) return e;
    const int64_t fb = (int64_t)a.H * a.W * sizeof(T);
    for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
        const int nb = (int)((batch - b0) < 65535 ? (batch - b0) : 65535);
        StagePlaneArgs ab = a;
        const int64_t off = b0 * fb;
        ab.u = static_cast<const char *>(a.u) + off;
        ab.f = static_cast<const char *>(a.f) + off;
        ab.p = static_cast<char *>(a.p) + off;
        if (a.w) ab.w = static_cast<char *>(a.w) + off;
        ab.u_out = static_cast<char *>(a.u_out) + off;
        dim3 g = grid0;
        g.z = nb;
        ka<<<g, PTHREADS, sa, st>>>(ab);
        kb<<<g, PTHREADS, sb, st>>>(ab);
    }
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_conv_plane(const ConvPlaneArgs &a, int64_t batch, cudaStream_t st) {
    const size_t sm = a.h.nt * sizeof(PlaneTap) +
                      (size_t)(PT + a.h.ht + a.h.hb) * (PT + a.h.hl + a.h.hr + 1) * sizeof(T);
    cudaError_t e = func_smem_attr((const void *)k_conv_plane<T>, sm);
    if (e != cudaSuccess) return e;
    const int64_t fb = (int64_t)a.H * a.W * sizeof(T);
    for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
        const int nb = (int)((batch - b0) < 65535 ? (batch - b0) : 65535);
        ConvPlaneArgs ab = a;
        ab.in = static_cast<const char *>(a.in) + b0 * fb;
        ab.out = static_cast<char *>(a.out) + b0 * fb;
        k_conv_plane<T><<<dim3((a.W + PT - 1) / PT, (a.H + PT - 1) / PT, nb), PTHREADS, sm, st>>>(ab);
    }
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_diffusion(const void *u, void *out, int64_t batch, int H, int W, double eps_r2, cudaStream_t st) {
    const int64_t fb = (int64_t)H * W * sizeof(T);
    for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
        const int nb = (int)((batch - b0) < 65535 ? (batch - b0) : 65535);
        k_diffusion<T><<<dim3((W + PT - 1) / PT, (H + PT - 1) / PT, nb), PTHREADS, 0, st>>>(
            reinterpret_cast<const T *>(static_cast<const char *>(u) + b0 * fb),
            reinterpret_cast<T *>(static_cast<char *>(out) + b0 * fb), H, W, T(eps_r2));
    }
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_robust_weight(const void *f, const void *b, void *out, int64_t n, double eps2, double floor,
                                 int floored, const LutView &lut, cudaStream_t st) {
    k_robust_weight<T><<<ew_blocks(n), 256, 0, st>>>(static_cast<const T *>(f), static_cast<const T *>(b),
                                                     static_cast<T *>(out), n, T(eps2), T(floor), floored, lut);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_lut_r1(const void *x, void *out, int64_t n, const LutView &lut, cudaStream_t st) {
    if (sizeof(T) == 8)
        k_lut_r1_ref<<<ew_blocks(n), 256, 0, st>>>(static_cast<const double *>(x), static_cast<double *>(out), n, lut);
    else
        k_lut_r1<T><<<ew_blocks(n), 256, 0, st>>>(static_cast<const T *>(x), static_cast<T *>(out), n, lut);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_ratio(const void *f, const void *b, const void *w, void *out, int64_t n, cudaStream_t st) {
    k_ratio<T><<<ew_blocks(n), 256, 0, st>>>(static_cast<const T *>(f), static_cast<const T *>(b),
                                             static_cast<const T *>(w), static_cast<T *>(out), n);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_combine(const void *u, const void *num, const void *den, const void *d, void *out, int64_t n,
                           double alpha, cudaStream_t st) {
    k_combine<T><<<ew_blocks(n), 256, 0, st>>>(static_cast<const T *>(u), static_cast<const T *>(num),
                                               static_cast<const T *>(den), static_cast<const T *>(d),
                                               static_cast<T *>(out), n, T(alpha));
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_guard(void *x, int64_t n, cudaStream_t st) {
    k_guard<T><<<ew_blocks(n), 256, 0, st>>>(static_cast<T *>(x), n);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_min(const void *x, int64_t n, double *partial, int nblocks, cudaStream_t st) {
    k_min_partial<T><<<nblocks, 256, 0, st>>>(static_cast<const T *>(x), n, partial);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_convert(const void *in, void *out, int64_t n, int to_double, cudaStream_t st) {
    k_convert<T><<<ew_blocks(n), 256, 0, st>>>(in, out, n, to_double);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_convert_in(const void *in, int in_type, void *out, int64_t n, cudaStream_t st) {
    k_convert_in<T><<<ew_blocks(n), 256, 0, st>>>(in, in_type, static_cast<T *>(out), n);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_convert_out(const void *in, void *out, int out_type, int64_t n, cudaStream_t st) {
    k_convert_out<T><<<ew_blocks(n), 256, 0, st>>>(static_cast<const T *>(in), out, out_type, n);
    return cudaGetLastError();
}

#define MD_INST(T)                                                                                      \
    template cudaError_t launch_stage_plane<T>(const StagePlaneArgs &, bool, int64_t, cudaStream_t);     \
    template cudaError_t launch_conv_plane<T>(const ConvPlaneArgs &, int64_t, cudaStream_t);             \
    template cudaError_t launch_diffusion<T>(const void *, void *, int64_t, int, int, double, cudaStream_t); \
    template cudaError_t launch_robust_weight<T>(const void *, const void *, void *, int64_t, double,   \
                                                 double, int, const LutView &, cudaStream_t);           \
    template cudaError_t launch_ratio<T>(const void *, const void *, const void *, void *, int64_t,     \
                                         cudaStream_t);                                                 \
    template cudaError_t launch_combine<T>(const void *, const void *, const void *, const void *,      \
                                           void *, int64_t, double, cudaStream_t);                      \
    template cudaError_t launch_guard<T>(void *, int64_t, cudaStream_t);                                \
    template cudaError_t launch_lut_r1<T>(const void *, void *, int64_t, const LutView &, cudaStream_t); \
    template cudaError_t launch_min<T>(const void *, int64_t, double *, int, cudaStream_t);             \
    template cudaError_t launch_convert<T>(const void *, void *, int64_t, int, cudaStream_t);          \
    template cudaError_t launch_convert_in<T>(const void *, int, void *, int64_t, cudaStream_t);       \
    template cudaError_t launch_convert_out<T>(const void *, void *, int, int64_t, cudaStream_t);
MD_INST(double)
MD_INST(float)
#undef MD_INST

}  // namespace md
