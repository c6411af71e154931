// md_plane_fast.cu -- register-blocked direct 2D convolution stages of one RRRL iteration
// for 2D PSFs (FOURIER_2D with direct periodic taps, or the clamped spatial convolver).
//
// Replaces _FourierConvolver2D / _SpatialConvolver inside _iterate_rrrl (deconv.py:295-307,
// 359-376, 512-521) together with _weight_arrays (142-162), _diffusion_arrays (187-213) and
// _combine (421-446).
//
// Tile 64 x 32 outputs per block, 256 threads; thread (row ty, column group cx) owns the 8
// outputs x = cx + 8 r (r = 0..7) of row ty, so a warp's lanes read consecutive shared-memory
// words for every tap. The tap list lives in the kernel parameters as (smem offset, weight)
// pairs precomputed on the host for the tile stride, so a tap costs one offset add, eight
// shared loads with immediate offsets and eight FMAs, shared by the eight outputs.
#include "md_plane.h"
#include "md_plane_fast.h"
#include "md_linefast.cuh"

namespace md {

constexpr int FX = 64, FY = 32;           // output tile
constexpr int FR = 8;                     // outputs per thread (stride 8 along x)

__device__ __forceinline__ int pf_resolve(int k, int n, int periodic) {
    // halos never exceed the extent, so one conditional wrap suffices (no integer modulo)
    if (periodic) return k < 0 ? k + n : (k >= n ? k - n : k);
    return k < 0 ? 0 : (k >= n ? n - 1 : k);
}

template <typename T>
__device__ void pf_load(T *s, int ss, const T *__restrict__ src, int H, int W, int y0, int x0, const PlaneHalo &h,
                        int periodic, int slab) {
    const int rows = FY + h.ht + h.hb, cols = FX + h.hl + h.hr;
    for (int i = threadIdx.x / 32; i < rows; i += blockDim.x / 32) {
        // slab mode: the caller's buffer carries the neighbours' rows (halo), read them as is
        const int y = slab ? y0 - h.ht + i : pf_resolve(y0 - h.ht + i, H, periodic);
        const T *srow = src + (int64_t)y * W;
        for (int j = threadIdx.x & 31; j < cols; j += 32) s[i * ss + j] = srow[pf_resolve(x0 - h.hl + j, W, periodic)];
    }
}

template <typename T, int MAXT>
__device__ __forceinline__ void pf_taps(const T *s, const FastTaps<T, MAXT> &tp, T acc[FR]) {
#pragma unroll
    for (int r = 0; r < FR; ++r) acc[r] = T(0);
    for (int t = 0; t < tp.nt; ++t) {
        const T *p = s + tp.off[t];
        const T w = tp.w[t];
#pragma unroll
        for (int r = 0; r < FR; ++r) acc[r] += w * p[8 * r];
    }
}

// num and den of the adjoint pair share the tap decode (deconv.py:425-430: adjoint_pair)
template <typename T, int MAXT>
__device__ __forceinline__ void pf_taps2(const T *s0, const T *s1, const FastTaps<T, MAXT> &tp, T a0[FR], T a1[FR]) {
#pragma unroll
    for (int r = 0; r < FR; ++r) a0[r] = a1[r] = T(0);
    const int d = (int)(s1 - s0);
    for (int t = 0; t < tp.nt; ++t) {
        const T *p = s0 + tp.off[t];
        const T w = tp.w[t];
#pragma unroll
        for (int r = 0; r < FR; ++r) {
            a0[r] += w * p[8 * r];
            a1[r] += w * p[d + 8 * r];
        }
    }
}

template <typename T, int MAXT, bool ROBUST>
__global__ void __launch_bounds__(256)
k_plane_a_fast(PlaneFastArgs<T, MAXT> a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T *su = reinterpret_cast<T *>(smem_raw);
    const int H = a.H, W = a.W;
    const int64_t fsz = (int64_t)H * W;
    const int64_t fr = blockIdx.z;
    const T *u = a.u + fr * fsz;
    const T *f = a.f + fr * fsz;
    T *p = a.p + fr * fsz;
    T *w = a.w + fr * fsz;
    const int y0 = blockIdx.y * FY, x0 = blockIdx.x * FX;
    const int ss = FX + a.hb.hl + a.hb.hr + 1;
    pf_load<T>(su, ss, u, H, W, y0, x0, a.hb, a.periodic, a.slab);
    __syncthreads();
    const int ty = threadIdx.x >> 3, cx = threadIdx.x & 7;
    const int y = y0 + ty;
    if (y >= H) return;
    // observation first: loads issued after the p / W stores below would wait for them
    T fr8[FR];
#pragma unroll
    for (int r = 0; r < FR; ++r) {
        const int x = x0 + cx + 8 * r;
        fr8[r] = x < W ? f[(int64_t)y * W + x] : T(1);
    }
    T b[FR];
    pf_taps<T, MAXT>(su + (ty + a.hb.ht) * ss + a.hb.hl + cx, a.tb, b);
    const T eps_d2 = a.eps_d2;
#pragma unroll
    for (int r = 0; r < FR; ++r) {
        const int x = x0 + cx + 8 * r;
        if (x >= W) continue;
        const int64_t o = (int64_t)y * W + x;
        const T bb = b[r] > T(kGuard) ? b[r] : T(kGuard);
        const T fv = fr8[r];
        const T ratio = fv * frcp(bb);
        if (ROBUST) {
            const T wv = T(0.5) * frsqrt(r1_fast<T>(a.lut, bb * frcp(fv)) * fv + eps_d2);
            w[o] = wv;
            p[o] = wv * ratio;
        } else {
            p[o] = ratio;
        }
    }
}

template <typename T, int MAXT, bool ROBUST>
__global__ void __launch_bounds__(256)
k_plane_b_fast(PlaneFastArgs<T, MAXT> a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int H = a.H, W = a.W;
    const int ss = FX + a.ha.hl + a.ha.hr + 1;
    const int rows = FY + a.ha.ht + a.ha.hb;
    T *sp = reinterpret_cast<T *>(smem_raw);
    T *sw = sp + rows * ss;
    T *su = ROBUST ? sw + rows * ss : sw;          // (FY+4) x (FX+5): u with a 2-pixel halo
    constexpr int US = FX + 5;
    T *sg = su + (FY + 4) * US;                     // (FY+2) x (FX+3): diffusivity
    constexpr int GS = FX + 3;
    const int64_t fsz = (int64_t)H * W;
    const int64_t fr = blockIdx.z;
    const T *u = a.u + fr * fsz;
    T *uo = a.u_out + fr * fsz;
    const int y0 = blockIdx.y * FY, x0 = blockIdx.x * FX;
    pf_load<T>(sp, ss, a.p + fr * fsz, H, W, y0, x0, a.ha, a.periodic, a.slab);
    if (ROBUST) pf_load<T>(sw, ss, a.w + fr * fsz, H, W, y0, x0, a.ha, a.periodic, a.slab);
    const int gy0 = a.gy0, Hg = a.Hg;
    for (int i = threadIdx.x / 32; i < FY + 4; i += 8) {
        const int yy = y0 - 2 + i;
        const bool rok = gy0 + yy >= 0 && gy0 + yy < Hg && (a.slab || (yy >= 0 && yy < H));
        for (int j = threadIdx.x & 31; j < FX + 4; j += 32) {
            const int xx = x0 - 2 + j;
            su[i * US + j] = (rok && xx >= 0 && xx < W) ? u[(int64_t)yy * W + xx] : T(0);
        }
    }
    __syncthreads();
    const T eps_r2 = a.eps_r2;
    if (a.has_d) {
        for (int i = threadIdx.x / 32; i < FY + 2; i += 8) {
            const int yy = y0 - 1 + i;
            const int gyy = gy0 + yy;
            if (gyy < 0 || gyy >= Hg) continue;
            for (int j = threadIdx.x & 31; j < FX + 2; j += 32) {
                const int xx = x0 - 1 + j;
                if (xx < 0 || xx >= W) continue;
                const T *c = su + (i + 1) * US + (j + 1);
                const T c0 = c[0];
                T q = T(0);
                if (xx + 1 < W) { const T d = c[1] - c0; q += d * d; }
                if (xx > 0) { const T d = c0 - c[-1]; q += d * d; }
                if (gyy + 1 < Hg) { const T d = c[US] - c0; q += d * d; }
                if (gyy > 0) { const T d = c0 - c[-US]; q += d * d; }
                sg[i * GS + j] = T(0.5) * frsqrt(T(0.5) * q + eps_r2);
            }
        }
        __syncthreads();
    }
    const int ty = threadIdx.x >> 3, cx = threadIdx.x & 7;
    const int y = y0 + ty;
    if (y >= H) return;
    T num[FR], den[FR];
    if (ROBUST) {
        pf_taps2<T, MAXT>(sp + (ty + a.ha.ht) * ss + a.ha.hl + cx, sw + (ty + a.ha.ht) * ss + a.ha.hl + cx, a.ta,
                          num, den);
    } else {
        pf_taps<T, MAXT>(sp + (ty + a.ha.ht) * ss + a.ha.hl + cx, a.ta, num);
    }
    const T alpha = a.alpha;
#pragma unroll
    for (int r = 0; r < FR; ++r) {
        const int tx = cx + 8 * r;
        const int x = x0 + tx;
        if (x >= W) continue;
        const T *c = su + (ty + 2) * US + (tx + 2);
        const T uv = c[0];
        T d = T(0);
        if (a.has_d) {
            const T *g = sg + (ty + 1) * GS + (tx + 1);
            const T gc = g[0];
            if (x + 1 < W) d += (gc + g[1]) * (c[1] - uv);
            if (x > 0) d -= (g[-1] + gc) * (uv - c[-1]);
            if (gy0 + y + 1 < Hg) d += (gc + g[GS]) * (c[US] - uv);
            if (gy0 + y > 0) d -= (g[-GS] + gc) * (uv - c[-US]);
        }
        T nm = num[r];
        T dn = ROBUST ? den[r] : T(1);
        if (a.has_d) {
            nm += alpha * (d > T(0) ? d : T(0));
            dn -= alpha * (d < T(0) ? d : T(0));
        } else if (!ROBUST) {
            uo[(int64_t)y * W + x] = uv * nm;
            continue;
        }
        dn = dn > T(kGuard) ? dn : T(kGuard);
        uo[(int64_t)y * W + x] = (uv * nm) * frcp(dn);
    }
}

// ---------------------------------------------------------------------------------- host

bool plane_fast_supported(const PlaneHalo &hb, const PlaneHalo &ha, int dtype) {
    if (hb.nt > kPlaneMaxTaps || ha.nt > kPlaneMaxTaps) return false;
    const size_t es = dtype == 0 ? 8 : 4;
    const size_t sa = (size_t)(FY + ha.ht + ha.hb) * (FX + ha.hl + ha.hr + 1);
    const size_t need = (2 * sa + (FY + 4) * (FX + 5) + (FY + 2) * (FX + 3)) * es;
    return need <= 200 * 1024;
}

template <typename T, int MAXT>
static void fill_fast_taps(FastTaps<T, MAXT> &ft, const std::vector<PlaneTap> &taps, int ss) {
    ft.nt = (int)taps.size();
    for (int t = 0; t < ft.nt; ++t) {
        ft.off[t] = taps[t].dy * ss + taps[t].dx;
        ft.w[t] = T(taps[t].w);
    }
}

template <typename T>
cudaError_t launch_plane_fast(const PlaneFastDesc &d, bool robust, int64_t batch, cudaStream_t st) {
    constexpr int MAXT = kPlaneMaxTaps;
    PlaneFastArgs<T, MAXT> a{};
    a.u = static_cast<const T *>(d.u);
    a.f = static_cast<const T *>(d.f);
    a.p = static_cast<T *>(d.p);
    a.w = static_cast<T *>(d.w);
    a.u_out = static_cast<T *>(d.u_out);
    a.H = d.H; a.W = d.W; a.periodic = d.periodic;
    a.slab = d.slab; a.gy0 = d.slab ? d.gy0 : 0; a.Hg = d.slab ? d.Hg : d.H;
    a.hb = d.hb; a.ha = d.ha;
    fill_fast_taps<T, MAXT>(a.tb, *d.taps_blur, FX + d.hb.hl + d.hb.hr + 1);
    fill_fast_taps<T, MAXT>(a.ta, *d.taps_adj, FX + d.ha.hl + d.ha.hr + 1);
    a.alpha = T(d.alpha); a.eps_d2 = T(d.eps_d2); a.eps_r2 = T(d.eps_r2); a.has_d = d.has_d;
    a.lut = d.lut;
    const size_t sa = (size_t)(FY + d.hb.ht + d.hb.hb) * (FX + d.hb.hl + d.hb.hr + 1) * sizeof(T);
    const size_t tb = (size_t)(FY + d.ha.ht + d.ha.hb) * (FX + d.ha.hl + d.ha.hr + 1);
    const size_t sb = ((robust ? 2 : 1) * tb + (FY + 4) * (FX + 5) + (FY + 2) * (FX + 3)) * sizeof(T);
    auto ka = robust ? k_plane_a_fast<T, MAXT, true> : k_plane_a_fast<T, MAXT, false>;
    auto kb = robust ? k_plane_b_fast<T, MAXT, true> : k_plane_b_fast<T, MAXT, false>;
    cudaError_t e = cudaFuncSetAttribute(ka, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sa);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb);
    if (e != cudaSuccess) return e;
    if (d.slab) {
        // stage A over the extended rows [row_a0, row_a0 + rows_a), stage B over the own rows
        PlaneFastArgs<T, MAXT> aa = a;
        const int64_t off = (int64_t)d.row_a0 * d.W;
        aa.u += off; aa.f += off; aa.p += off; aa.w += off;
        aa.H = d.rows_a; aa.gy0 = d.gy0 + d.row_a0;
        ka<<<dim3((d.W + FX - 1) / FX, (d.rows_a + FY - 1) / FY, 1), 256, sa, st>>>(aa);
        kb<<<dim3((d.W + FX - 1) / FX, (d.H + FY - 1) / FY, 1), 256, sb, st>>>(a);
        return cudaGetLastError();
    }
    const int64_t fsz = (int64_t)d.H * d.W;
    for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
        const int nb = (int)((batch - b0) < 65535 ? (batch - b0) : 65535);
        PlaneFastArgs<T, MAXT> ab = a;
        ab.u += b0 * fsz; ab.f += b0 * fsz; ab.p += b0 * fsz; ab.w += b0 * fsz; ab.u_out += b0 * fsz;
        const dim3 grid((d.W + FX - 1) / FX, (d.H + FY - 1) / FY, nb);
        ka<<<grid, 256, sa, st>>>(ab);
        kb<<<grid, 256, sb, st>>>(ab);
    }
    return cudaGetLastError();
}

template cudaError_t launch_plane_fast<double>(const PlaneFastDesc &, bool, int64_t, cudaStream_t);
template cudaError_t launch_plane_fast<float>(const PlaneFastDesc &, bool, int64_t, cudaStream_t);

}  // namespace md
