// md_plane_fast.cu -- register-blocked direct 2D convolution stages of one RRRL iteration
// for 2D PSFs (FOURIER_2D with direct periodic taps, or the clamped spatial convolver).
//
// Replaces _FourierConvolver2D / _SpatialConvolver inside _iterate_rrrl (deconv.py:295-307,
// 359-376, 512-521) together with _weight_arrays (142-162), _diffusion_arrays (187-213) and
// _combine (421-446).
//
// Tile 64 x 32 outputs per block, 256 threads; thread (row group tp, column cx) owns the
// outputs of rows PR tp .. PR tp + PR-1 at x = cx + PX r (round 2: PR = 4 rows x 2 columns at
// stride 32, a warp reads 32 consecutive shared-memory elements per tap; round 1: row pairs x 4
// columns at stride 16). Taps are regrouped on the host into columns (md_coltaps.cuh): each
// loaded value feeds all PR rows. Stage B stages p and W interleaved, so one load feeds both
// halves of the adjoint pair.
#include "md_plane.h"
#include "md_plane_fast.h"
#include "md_linefast.cuh"
#include "md_tma.cuh"

#include <algorithm>
#include <cstdlib>

namespace md {

constexpr int FX = 64, FY = 32;           // output tile
#ifndef MD_PLANE_ROWS
#define MD_PLANE_ROWS 4
#endif
// thread = PR consecutive output rows x PJ columns at stride PX (256 threads cover the tile):
// PR = 4 rows cost len + 3 shared loads per tap column for 4 rows, the row pair len + 1 for 2
// (md_coltaps.cuh); the sums, and so the results, are the same
#ifndef MD_PLANE_ROWS_B
#define MD_PLANE_ROWS_B MD_PLANE_ROWS
#endif
template <int R> struct PlaneMap {
    static constexpr int PR = R;
    static constexpr int PJ = 8 / R;           // outputs per row per thread
    static constexpr int PX = FX / PJ;         // their column stride (= the threads per row)
    static_assert(PR * PJ == 8 && (FY / PR) * PX == 256, "tile / thread mapping");
};
constexpr int PS = 72;                    // u / g tile stride: 2 * PS = 16 (mod 32) -> half-warps on disjoint banks

__device__ __forceinline__ int pf_resolve(int k, int n, int periodic) {
    // a tile (64 x 32 plus halos) may be wider / taller than a small frame, so positions can lie
    // more than one extent outside: a full wrap (resolved once per tile column / row, not per
    // element). Found by the checked build: a 32-wide frame read past its buffer with the
    // single conditional wrap this replaced.
    if (periodic) {
        k = k < 0 ? k + n : (k >= n ? k - n : k);          // the common case: within one extent
        if ((unsigned)k >= (unsigned)n) {                   // small frames: a full wrap
            k %= n;
            k = k < 0 ? k + n : k;
        }
        return k;
    }
    return k < 0 ? 0 : (k >= n ? n - 1 : k);
}

// tile rows [y0 - ht, y0 + FY + hb) x cols [x0 - hl, x0 + FX + hr) of one or two fields. A warp
// walks rows, its lanes the columns (CJ column slots per lane, resolved once per block, so
// no per-element division or wrap); two rows per step keep 2 CJ global loads in flight.
constexpr int PF_CJ = 4;                  // cols <= 32 * PF_CJ (FX + x-halos <= 128)
#ifndef MD_PLANE_CP_ASYNC
#define MD_PLANE_CP_ASYNC 1
#endif
#ifndef MD_PLANE_TMA
#define MD_PLANE_TMA 1             // u tiles by TMA (md_tma.cuh) in whole-frame launches
#endif
template <typename T, typename E, typename Get>
__device__ void pf_load(E *s, int ss, int H, int W, int y0, int x0, const PlaneHalo &h, int periodic, int slab,
                        int ylo, int yhi, Get get) {
    const int rows = FY + h.ht + h.hb, cols = FX + h.hl + h.hr;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    int xr[PF_CJ];
#pragma unroll
    for (int c = 0; c < PF_CJ; ++c) {
        const int j = lane + 32 * c;
        xr[c] = j < cols ? pf_resolve(x0 - h.hl + j, W, periodic) : -1;
    }
    auto yres = [&](int i) {
        // slab mode: the caller's buffer carries the neighbours' rows (halo), read them as is; the
        // last tile row band may reach past the halo (rows_a is not a multiple of FY): those rows
        // only feed outputs that are not stored, so they read the nearest existing row
        const int y = y0 - h.ht + i;
        MD_CHECK(!slab || ylo < yhi);
        return slab ? (y < ylo ? ylo : (y >= yhi ? yhi - 1 : y)) : pf_resolve(y, H, periodic);
    };
    for (int i = warp; i < rows; i += 2 * nw) {
        const int i2 = i + nw;
        const bool two = i2 < rows;
        const int64_t b0 = (int64_t)yres(i) * W, b1 = two ? (int64_t)yres(i2) * W : b0;
        E v0[PF_CJ], v1[PF_CJ];
#pragma unroll
        for (int c = 0; c < PF_CJ; ++c) {
            if (xr[c] >= 0) {
                v0[c] = get(b0 + xr[c]);
                if (two) v1[c] = get(b1 + xr[c]);
            }
        }
#pragma unroll
        for (int c = 0; c < PF_CJ; ++c) {
            if (xr[c] >= 0) {
                s[i * ss + lane + 32 * c] = v0[c];
                if (two) s[i2 * ss + lane + 32 * c] = v1[c];
            }
        }
    }
}

// the same tile of up to two fields, loaded with cp.async (LDGSTS: global -> shared without a
// register round trip, every element of the tile in flight at once) -- field a into the first
// element of each E slot, field b (optional) into the second. Caller: cp_async_wait_all() and
// __syncthreads() before use.
__device__ __forceinline__ void cp_async_elem(void *dst, const void *src, int bytes) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
    if (bytes == 16) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
    else if (bytes == 8) asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
    else asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// fpair (optional, E = the pair type): the two fields interleaved in one array -- one copy of
// sizeof(E) bytes per element instead of two
template <typename T, typename E>
__device__ void pf_load_async(E *s, int ss, int H, int W, int y0, int x0, const PlaneHalo &h, int periodic, int slab,
                              int ylo, int yhi, const T *fa, const T *fb, const E *fpair = nullptr) {
    const int rows = FY + h.ht + h.hb, cols = FX + h.hl + h.hr;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    int xr[PF_CJ];
#pragma unroll
    for (int c = 0; c < PF_CJ; ++c) {
        const int j = lane + 32 * c;
        xr[c] = j < cols ? pf_resolve(x0 - h.hl + j, W, periodic) : -1;
    }
    for (int i = warp; i < rows; i += nw) {
        const int y = y0 - h.ht + i;
        const int yy = slab ? (y < ylo ? ylo : (y >= yhi ? yhi - 1 : y)) : pf_resolve(y, H, periodic);
        const int64_t b = (int64_t)yy * W;
#pragma unroll
        for (int c = 0; c < PF_CJ; ++c) {
            if (xr[c] < 0) continue;
            if (fpair) {
                cp_async_elem(s + i * ss + lane + 32 * c, fpair + b + xr[c], (int)sizeof(E));
                continue;
            }
            T *d = reinterpret_cast<T *>(s + i * ss + lane + 32 * c);
            cp_async_elem(d, fa + b + xr[c], (int)sizeof(T));
            if (fb) cp_async_elem(d + 1, fb + b + xr[c], (int)sizeof(T));
        }
    }
}

// Stage A's u tile in shared memory, laid out for TMA: a box must start on a 16-byte column
// boundary (measured: an unaligned inner start coordinate is an illegal instruction), so the
// tile row starts at column xoff = (-hl) mod (16 / sizeof(T)) of an smem row of pf_stride_a
// elements (a multiple of 16 bytes, >= xoff + the tile width); x0 is a multiple of 64, so xoff
// is the same for every tile of a launch. (A warp reads 32 consecutive columns of one row: any
// stride is conflict-free.)
template <typename T> __host__ __device__ inline int pf_xoff_a(const PlaneHalo &h) {
    constexpr int g = 16 / (int)sizeof(T);
    return ((-h.hl) % g + g) % g;
}
template <typename T> __host__ __device__ inline int pf_stride_a(const PlaneHalo &h) {
    constexpr int g = 16 / (int)sizeof(T);
    const int need = FX + h.hl + h.hr + pf_xoff_a<T>(h);
    return (need + g - 1) / g * g;
}
// stage B's u tile (columns x0-2 ..): the same rule, a constant offset for float
template <typename T> constexpr int pf_xoff_b() { return sizeof(T) == 4 ? 2 : 0; }
// stage B's (p, W) pair tile: pairs of 16 (float64) / 8 (float32) bytes, the same rule
template <typename T> __host__ __device__ inline int pf_xoff_pw(const PlaneHalo &h) {
    constexpr int g = 16 / (2 * (int)sizeof(T));
    return ((-h.hl) % g + g) % g;
}
template <typename T> __host__ __device__ inline int pf_stride_b(const PlaneHalo &h) {
    constexpr int g = 16 / (2 * (int)sizeof(T));
    const int need = FX + h.hl + h.hr + pf_xoff_pw<T>(h);
    return (need + g - 1) / g * g;
}

#ifndef MD_PLANE_A_MINB
#define MD_PLANE_A_MINB 4          // <= 64 registers: 4 blocks per SM (the interleaved-store branch pushed it to 76 and 3)
#endif
template <typename T, bool ROBUST>
__global__ void __launch_bounds__(256, MD_PLANE_A_MINB)
k_plane_a_fast(PlaneFastArgs<T> a, const __grid_constant__ CUtensorMap tmu) {
    constexpr int PR = PlaneMap<MD_PLANE_ROWS>::PR, PJ = PlaneMap<MD_PLANE_ROWS>::PJ, PX = PlaneMap<MD_PLANE_ROWS>::PX;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T *su = reinterpret_cast<T *>(smem_raw);
    const int H = a.H, W = a.W;
    const int64_t fsz = (int64_t)H * W;
    const int64_t fr = blockIdx.z;
    const T *u = a.u + fr * fsz;
    const T *f = a.f + fr * fsz;
    T *p = a.p + fr * fsz;
    T *w = a.w + fr * fsz;
    const int y0 = blockIdx.y * FY, x0 = blockIdx.x * FX;
    const int ss = a.ssa;
    const int trows = FY + a.hb.ht + a.hb.hb;
    const int xo = pf_xoff_a<T>(a.hb);
    poison_smem(smem_raw);
    MD_CHECK((smem_addr_of(su) & 127) == 0 && (size_t)trows * ss * sizeof(T) + 8 <= dyn_smem_bytes() &&
             ((x0 - a.hb.hl - xo) * (int)sizeof(T)) % 16 == 0);
    T *st = su + xo;                                  // the tile's column 0 (x0 - hl)
    // interior tiles (no wrap / clamp inside the halo): one TMA box of trows x ss elements (the
    // padding columns past the halo read whatever lies there, or zeros past the frame)
    if (a.tma_a && x0 - a.hb.hl >= 0 && x0 + FX + a.hb.hr <= W && y0 - a.hb.ht >= 0 && y0 + FY + a.hb.hb <= H) {
        uint64_t *bar = reinterpret_cast<uint64_t *>((reinterpret_cast<uintptr_t>(su + trows * ss) + 7) & ~uintptr_t(7));
        if (threadIdx.x == 0) {
            tma_bar_arm(bar, (uint32_t)(trows * ss * sizeof(T)));
            tma_load_3d(su, &tmu, x0 - a.hb.hl - xo, y0 - a.hb.ht, (int)blockIdx.z, bar);
        }
        __syncthreads();                            // the barrier is initialised
        tma_bar_wait(bar);
    } else {
#if MD_PLANE_CP_ASYNC
        pf_load_async<T, T>(st, ss, H, W, y0, x0, a.hb, a.periodic, a.slab, a.ylo, a.yhi, u, nullptr);
        cp_async_wait_all();
#else
        pf_load<T>(st, ss, H, W, y0, x0, a.hb, a.periodic, a.slab, a.ylo, a.yhi, [&](int64_t o) { return u[o]; });
#endif
    }
    __syncthreads();
    const int tp = threadIdx.x / PX, cx = threadIdx.x % PX;
    const int yp = y0 + PR * tp;
    if (yp >= H) return;
    // observation first: loads issued after the p / W stores below would wait for them
    T fv[PR][PJ];
#pragma unroll
    for (int k = 0; k < PR; ++k)
#pragma unroll
        for (int r = 0; r < PJ; ++r) {
            const int x = x0 + cx + PX * r;
            fv[k][r] = (x < W && yp + k < H) ? f[(int64_t)(yp + k) * W + x] : T(1);
        }
    T b[PR][PJ];
    col_taps_rows<T, PR, PJ, PX>(st + (PR * tp + a.hb.ht) * ss + a.hb.hl + cx, ss, a.tb, b);
    const T eps_d2 = a.eps_d2;
#pragma unroll
    for (int k = 0; k < PR; ++k) {
        const int y = yp + k;
        if (y >= H) break;
#pragma unroll
        for (int r = 0; r < PJ; ++r) {
            const int x = x0 + cx + PX * r;
            if (x >= W) continue;
            const int64_t o = (int64_t)y * W + x;
            const T bb = dmax_sel(b[k][r], T(kGuard));
            const T ratio = fv[k][r] * frcp(bb);
            T pv = ratio, wv = T(0);
            if (ROBUST) {
                wv = T(0.5) * frsqrt(r1_fast<T>(a.lut, bb * frcp(fv[k][r])) * fv[k][r] + eps_d2);
                pv = wv * ratio;
            }
            if (a.pwi) {                              // interleaved (p, W): one store
                using T2 = typename Vec2<T>::type;
                T2 v;
                v.x = pv;
                v.y = wv;
                // parity-split rows (k_plane_b_adj): even columns, then odd ones
                const int64_t po = a.pw_split ? (int64_t)y * W + (x & 1) * (W >> 1) + (x >> 1) : o;
                reinterpret_cast<T2 *>(a.p)[fr * fsz + po] = v;
            } else {
                p[o] = pv;
                if (ROBUST) w[o] = wv;
            }
        }
    }
}

// MODE (shared layout, picked per launch in launch_plane_fast for the most blocks per SM):
//  0: (p, W) tile | u tile | diffusivity
//  1: (p, W) tile, the diffusivity computed after the column walk over it | u tile
//  2: (p, W) tile only: after the walk the u tile is loaded, and the diffusivity computed, over it
template <typename T, bool ROBUST, int MODE>
__global__ void __launch_bounds__(256)
k_plane_b_fast(PlaneFastArgs<T> a, const __grid_constant__ CUtensorMap tmu, const __grid_constant__ CUtensorMap tmpw) {
    constexpr int PR = PlaneMap<MD_PLANE_ROWS_B>::PR, PJ = PlaneMap<MD_PLANE_ROWS_B>::PJ, PX = PlaneMap<MD_PLANE_ROWS_B>::PX;
    using T2 = typename Vec2<T>::type;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int H = a.H, W = a.W;
    const int ss = a.ssb;
    const int rows = FY + a.ha.ht + a.ha.hb;
    T2 *spw = reinterpret_cast<T2 *>(smem_raw);
    const size_t pw_bytes = (rows * ss * sizeof(T2) + 127) & ~size_t(127);
    // (FY+4) x PS: u with a 2-pixel halo, 128-byte aligned (a TMA destination)
    T *su_box = reinterpret_cast<T *>(smem_raw + (MODE == 2 ? 0 : pw_bytes));
    T *su = su_box + pf_xoff_b<T>();                 // column 0 = x0 - 2 (TMA boxes start 16-byte aligned)
    // (FY+2) x PS: diffusivity
    T *sg = MODE == 0 ? su_box + (FY + 4) * PS : (MODE == 1 ? reinterpret_cast<T *>(smem_raw) : su_box + (FY + 4) * PS);
    unsigned char *end = MODE == 0 ? reinterpret_cast<unsigned char *>(sg + (FY + 2) * PS)
                                   : (MODE == 1 ? reinterpret_cast<unsigned char *>(su_box + (FY + 4) * PS) : smem_raw + pw_bytes);
    uint64_t *bar = reinterpret_cast<uint64_t *>((reinterpret_cast<uintptr_t>(end) + 7) & ~uintptr_t(7));
    uint64_t *bar2 = bar + 1;                        // MODE 2: the late u tile
    const int64_t fsz = (int64_t)H * W;
    const int64_t fr = blockIdx.z;
    const T *u = a.u + fr * fsz;
    T *uo = a.u_out + fr * fsz;
    const int y0 = blockIdx.y * FY, x0 = blockIdx.x * FX;
    const int xpw = pf_xoff_pw<T>(a.ha);
    T2 *sp = spw + xpw;                              // the (p, W) tile's column 0 (x0 - hl)
    poison_smem(smem_raw);
    MD_CHECK((smem_addr_of(spw) & 127) == 0 && (smem_addr_of(su_box) & 127) == 0 &&
             (size_t)(reinterpret_cast<unsigned char *>(bar + (MODE == 2 ? 2 : 1)) - smem_raw) <= dyn_smem_bytes() &&
             (MODE != 2 || reinterpret_cast<unsigned char *>(sg + (FY + 2) * PS) <= smem_raw + pw_bytes) &&
             ((x0 - a.ha.hl - xpw) * 2 * (int)sizeof(T)) % 16 == 0 && ((x0 - 2 - pf_xoff_b<T>()) * (int)sizeof(T)) % 16 == 0);
    // interleaved (p, W) and an interior tile: the whole pair tile as one TMA box (rows x ss
    // pairs, started on a 16-byte boundary); otherwise per element (wrap / clamp at the edges)
    const bool pw_tma = a.tma_pw && x0 - a.ha.hl >= 0 && x0 + FX + a.ha.hr <= W && y0 - a.ha.ht >= 0 &&
                        y0 + FY + a.ha.hb <= H;
    if (!pw_tma) {
        const T *pp = a.p + fr * fsz, *ww = a.w + fr * fsz;
        const T2 *ppw = a.pwi ? reinterpret_cast<const T2 *>(a.p) + fr * fsz : nullptr;
        // (p, W) tile by cp.async: issued here, in flight while the u tile loads below
        pf_load_async<T, T2>(sp, ss, H, W, y0, x0, a.ha, a.periodic, a.slab, a.ylo, a.yhi, pp, ROBUST ? ww : nullptr, ppw);
    }
    const int gy0 = a.gy0, Hg = a.Hg;
    // u with a 2-pixel halo (zero outside the frame / slab): one TMA box (whole-frame launches,
    // the map's zero fill = the zero halo) or cp.async with zero-fill
    auto load_u = [&](bool tma_issued) {
        if (!a.tma_b) {
            constexpr int UC = FX + 4;
            const int n = (FY + 4) * UC;
            for (int idx = threadIdx.x; idx < n; idx += blockDim.x) {
                const int i = idx / UC, j = idx - i * UC;
                const int yy = y0 - 2 + i, xx = x0 - 2 + j;
                const bool ok = gy0 + yy >= 0 && gy0 + yy < Hg && (a.slab ? (yy >= a.ylo && yy < a.yhi) : (yy >= 0 && yy < H)) &&
                                xx >= 0 && xx < W;
                const uint32_t d = (uint32_t)__cvta_generic_to_shared(su + i * PS + j);
                const T *src = ok ? u + (int64_t)yy * W + xx : u;
                if (sizeof(T) == 8)
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(ok ? 8 : 0) : "memory");
                else
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(src), "r"(ok ? 4 : 0) : "memory");
            }
        }
        (void)tma_issued;
    };
    if (threadIdx.x == 0 && ((MODE != 2 && a.tma_b) || pw_tma)) {
        // TMA boxes on one barrier: u (FY+4) x PS at (x0-2, y0-2), positions outside the frame
        // arriving as zeros (whole-frame launches only: a slab reads its halo rows as they are);
        // the (p, W) pairs as 2 ss elements per row
        const bool ub = MODE != 2 && a.tma_b;
        tma_bar_arm(bar, (uint32_t)((ub ? (FY + 4) * PS * sizeof(T) : 0) + (pw_tma ? rows * ss * sizeof(T2) : 0)));
        if (ub) tma_load_3d(su_box, &tmu, x0 - 2 - pf_xoff_b<T>(), y0 - 2, (int)blockIdx.z, bar);
        if (pw_tma) tma_load_3d(spw, &tmpw, 2 * (x0 - a.ha.hl - xpw), y0 - a.ha.ht, (int)blockIdx.z, bar);
    }
    if (MODE != 2) load_u(false);
    cp_async_wait_all();
    __syncthreads();                                 // (also: the TMA barrier is initialised)
    if ((MODE != 2 && a.tma_b) || pw_tma) {
        tma_bar_wait(bar);
        __syncthreads();
    }
    const T eps_r2 = a.eps_r2;
    auto diffusivity = [&]() {
        for (int i = threadIdx.x / 32; i < FY + 2; i += 8) {
            const int yy = y0 - 1 + i;
            const int gyy = gy0 + yy;
            if (gyy < 0 || gyy >= Hg) continue;
            for (int j = threadIdx.x & 31; j < FX + 2; j += 32) {
                const int xx = x0 - 1 + j;
                if (xx < 0 || xx >= W) continue;
                const T *c = su + (i + 1) * PS + (j + 1);
                const T c0 = c[0];
                T q = T(0);
                if (xx + 1 < W) { const T d = c[1] - c0; q += d * d; }
                if (xx > 0) { const T d = c0 - c[-1]; q += d * d; }
                if (gyy + 1 < Hg) { const T d = c[PS] - c0; q += d * d; }
                if (gyy > 0) { const T d = c0 - c[-PS]; q += d * d; }
                sg[i * PS + j] = T(0.5) * frsqrt(T(0.5) * q + eps_r2);
            }
        }
        __syncthreads();
    };
    const int tp = threadIdx.x / PX, cx = threadIdx.x % PX;
    const int ty0 = PR * tp;
    T2 nd[PR][PJ];
    if (MODE == 0) {
        if (a.has_d) diffusivity();
        if (y0 + ty0 >= H) return;
        col_taps_rows2<T, PR, PJ, PX>(sp + (ty0 + a.ha.ht) * ss + a.ha.hl + cx, ss, a.ta, nd);
    } else {
        const bool active = y0 + ty0 < H;
        if (active) col_taps_rows2<T, PR, PJ, PX>(sp + (ty0 + a.ha.ht) * ss + a.ha.hl + cx, ss, a.ta, nd);
        if (MODE == 2) {
            // the (p, W) tile is done with: the u tile over it, then the diffusivity behind it
            __syncthreads();
            if (threadIdx.x == 0 && a.tma_b) {
                // generic-proxy reads of this memory (the walk) before the async-proxy writes
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                tma_bar_arm(bar2, (uint32_t)((FY + 4) * PS * sizeof(T)));
                tma_load_3d(su_box, &tmu, x0 - 2 - pf_xoff_b<T>(), y0 - 2, (int)blockIdx.z, bar2);
            }
            load_u(true);
            cp_async_wait_all();
            __syncthreads();
            if (a.tma_b) {
                tma_bar_wait(bar2);
                __syncthreads();
            }
            if (a.has_d) diffusivity();
        } else if (a.has_d) {
            __syncthreads();                         // every warp is done with the (p, W) tile
            diffusivity();
        }
        if (!active) return;
    }
    const T alpha = a.alpha;
#pragma unroll
    for (int k = 0; k < PR; ++k) {
        const int ty = ty0 + k;
        const int y = y0 + ty;
        if (y >= H) break;
#pragma unroll
        for (int r = 0; r < PJ; ++r) {
            const int tx = cx + PX * r;
            const int x = x0 + tx;
            if (x >= W) continue;
            const T *c = su + (ty + 2) * PS + (tx + 2);
            const T uv = c[0];
            T d = T(0);
            if (a.has_d) {
                const T *g = sg + (ty + 1) * PS + (tx + 1);
                const T gc = g[0];
                if (x + 1 < W) d += (gc + g[1]) * (c[1] - uv);
                if (x > 0) d -= (g[-1] + gc) * (uv - c[-1]);
                if (gy0 + y + 1 < Hg) d += (gc + g[PS]) * (c[PS] - uv);
                if (gy0 + y > 0) d -= (g[-PS] + gc) * (uv - c[-PS]);
            }
            T nm = nd[k][r].x;
            T dn = ROBUST ? nd[k][r].y : T(1);
            if (a.has_d) {
                nm += alpha * dmax_sel(d, T(0));
                dn -= alpha * dmin_sel(d, T(0));
            } else if (!ROBUST) {
                uo[(int64_t)y * W + x] = uv * nm;
                continue;
            }
            dn = dmax_sel(dn, T(kGuard));
            uo[(int64_t)y * W + x] = (uv * nm) * frcp(dn);
        }
    }
}

// ------------------------------------------------ stage B, adjacent output columns (float64)
// (md_plane_fast.h AdjTaps): thread = 4 rows x 2 adjacent columns (warp = 4 rows of the 64-wide
// tile, lane l = columns 2l, 2l + 1); the (p, W) tile de-interleaved by column parity

// the pair tile [parity][rows][hh] per element (cp.async, 16 bytes): edge tiles (wrap / clamp),
// slabs (separate p / W fields) -- fpair: the parity-split pair field of stage A
template <typename T, typename E>
__device__ void pf_load_adj_async(E *s, int hh, int H, int W, int y0, int x0, int hle, const PlaneHalo &h,
                                  int periodic, int slab, int ylo, int yhi, const T *fa, const T *fb, const E *fpair) {
    const int rows = FY + h.ht + h.hb, cols = FX + hle + h.hr;
    const int half = (rows * hh + 7) & ~7;            // k_plane_b_adj's parity halves
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    int xr[PF_CJ], xs[PF_CJ];
#pragma unroll
    for (int c = 0; c < PF_CJ; ++c) {
        const int j = lane + 32 * c;
        xr[c] = j < cols ? pf_resolve(x0 - hle + j, W, periodic) : -1;
        xs[c] = xr[c] < 0 ? 0 : (xr[c] & 1) * (W >> 1) + (xr[c] >> 1);   // position in a split row
    }
    for (int i = warp; i < rows; i += nw) {
        const int y = y0 - h.ht + i;
        const int yy = slab ? (y < ylo ? ylo : (y >= yhi ? yhi - 1 : y)) : pf_resolve(y, H, periodic);
        const int64_t b = (int64_t)yy * W;
#pragma unroll
        for (int c = 0; c < PF_CJ; ++c) {
            if (xr[c] < 0) continue;
            const int j = lane + 32 * c;
            E *d = s + (j & 1) * half + i * hh + (j >> 1);
            if (fpair) {
                cp_async_elem(d, fpair + b + xs[c], (int)sizeof(E));
                continue;
            }
            T *dt = reinterpret_cast<T *>(d);
            cp_async_elem(dt, fa + b + xr[c], (int)sizeof(T));
            if (fb) cp_async_elem(dt + 1, fb + b + xr[c], (int)sizeof(T));
        }
    }
}

// 4 rows x 2 columns over one merged column of LEN steps, fully unrolled (the weights in registers)
template <typename T2, int LEN>
__device__ __forceinline__ void adj_walk_fixed(const T2 *p, int ss, const T2 *wc, T2 (&nd)[4][2]) {
    T2 w[LEN];
#pragma unroll
    for (int k = 0; k < LEN; ++k) w[k] = wc[k];
#pragma unroll
    for (int i = 0; i < LEN + 3; ++i) {
        const T2 v = p[i * ss];
#pragma unroll
        for (int r = 0; r < 4; ++r)
            if (i - r >= 0 && i - r < LEN) {
                const T2 wr = w[i - r];
                nd[r][0].x += wr.x * v.x;
                nd[r][0].y += wr.x * v.y;
                nd[r][1].x += wr.y * v.x;
                nd[r][1].y += wr.y * v.y;
            }
    }
}
// any length (the auto pick keeps this kernel to merged columns of <= 8 steps, which take the
// unrolled walks above; a weight window in registers here raised the kernel's register count)
template <typename T2>
__device__ __forceinline__ void adj_walk_any(const T2 *p, int ss, const T2 *wc, int len, T2 (&nd)[4][2]) {
    auto step = [&](const T2 &v, const T2 &wr, T2 (&o)[2]) {
        o[0].x += wr.x * v.x;
        o[0].y += wr.x * v.y;
        o[1].x += wr.y * v.x;
        o[1].y += wr.y * v.y;
    };
    for (int i = 0; i < len + 3; ++i) {
        const T2 v = p[i * ss];
#pragma unroll
        for (int r = 0; r < 4; ++r)
            if (i - r >= 0 && i - r < len) step(v, wc[i - r], nd[r]);
    }
}
template <typename T2, typename AT>
__device__ __forceinline__ void adj_walk(const T2 *s, int ss, const AT &tp, T2 (&nd)[4][2]) {
    for (int c = 0; c < tp.ncol; ++c) {
        const int2 ci = tp.c[c];
        const int len = ci.y & 0xffff;
        const T2 *wc = tp.w + (ci.y >> 16);
        const T2 *p = s + ci.x;
        switch (len) {
            case 1: adj_walk_fixed<T2, 1>(p, ss, wc, nd); break;
            case 2: adj_walk_fixed<T2, 2>(p, ss, wc, nd); break;
            case 3: adj_walk_fixed<T2, 3>(p, ss, wc, nd); break;
            case 4: adj_walk_fixed<T2, 4>(p, ss, wc, nd); break;
            case 5: adj_walk_fixed<T2, 5>(p, ss, wc, nd); break;
            case 6: adj_walk_fixed<T2, 6>(p, ss, wc, nd); break;
            case 7: adj_walk_fixed<T2, 7>(p, ss, wc, nd); break;
            case 8: adj_walk_fixed<T2, 8>(p, ss, wc, nd); break;
            default: adj_walk_any<T2>(p, ss, wc, len, nd);
        }
    }
}

// LATE: shared memory holds only the (p, W) tile; after the walk the u tile is loaded, and the
// diffusivity computed, over it (k_plane_b_fast's mode 2)
// B4: compiled for 4 blocks per SM (64 registers, a few spilled) -- the c4 wide line PSFs, whose
// late layout fits 4 blocks; otherwise for 3 (at most 80 registers: 84 would leave 2)
template <typename T, bool ROBUST, bool LATE, bool B4>
__global__ void __launch_bounds__(256, B4 ? 4 : 3)
k_plane_b_adj(PlaneFastArgs<T> a, const __grid_constant__ AdjTaps<T> t, const __grid_constant__ CUtensorMap tmu,
              const __grid_constant__ CUtensorMap tmpw) {
    static_assert(sizeof(T) == 8, "float64 only (the TV loads pair two columns in 16 bytes)");
    using T2 = typename Vec2<T>::type;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int H = a.H, W = a.W;
    const int hle = t.hle, hh = t.hh;
    const int rows = FY + a.ha.ht + a.ha.hb;
    // [parity][rows][hh] pairs; each half 128-byte aligned (a TMA destination)
    const int half = (rows * hh + 7) & ~7;
    T2 *spw = reinterpret_cast<T2 *>(smem_raw);
    const size_t pw_bytes = 2 * (size_t)half * sizeof(T2);
    T *su_box = reinterpret_cast<T *>(smem_raw + (LATE ? 0 : pw_bytes));
    T *su = su_box;                                  // column 0 = x0 - 2
    T *sg = su_box + (FY + 4) * PS;
    unsigned char *end = LATE ? smem_raw + pw_bytes : reinterpret_cast<unsigned char *>(sg + (FY + 2) * PS);
    uint64_t *bar = reinterpret_cast<uint64_t *>((reinterpret_cast<uintptr_t>(end) + 7) & ~uintptr_t(7));
    uint64_t *bar2 = bar + 1;
    const int64_t fsz = (int64_t)H * W;
    const int64_t fr = blockIdx.z;
    const T *u = a.u + fr * fsz;
    T *uo = a.u_out + fr * fsz;
    const int y0 = blockIdx.y * FY, x0 = blockIdx.x * FX;
    poison_smem(smem_raw);
    MD_CHECK((smem_addr_of(spw) & 127) == 0 && (smem_addr_of(su_box) & 127) == 0 && (hle & 1) == 0 &&
             2 * hh >= FX + hle + a.ha.hr && (W & 1) == 0 &&
             (!LATE || reinterpret_cast<unsigned char *>(sg + (FY + 2) * PS) <= smem_raw + pw_bytes) &&
             (size_t)(reinterpret_cast<unsigned char *>(bar + (LATE ? 2 : 1)) - smem_raw) <= dyn_smem_bytes());
    // interior tile of the parity-split pair field: two plain TMA boxes (the even and the odd
    // column pairs of the tile rows), each landing as [rows][hh]
    const bool pw_tma = a.tma_pw && x0 - hle >= 0 && ((x0 - hle) >> 1) + hh <= (W >> 1) && y0 - a.ha.ht >= 0 &&
                        y0 + FY + a.ha.hb <= H;
    if (!pw_tma) {
        const T *pp = a.p + fr * fsz, *ww = a.w + fr * fsz;
        const T2 *ppw = a.pwi ? reinterpret_cast<const T2 *>(a.p) + fr * fsz : nullptr;
        pf_load_adj_async<T, T2>(spw, hh, H, W, y0, x0, hle, a.ha, a.periodic, a.slab, a.ylo, a.yhi, pp,
                                 ROBUST ? ww : nullptr, ppw);
    }
    const int gy0 = a.gy0, Hg = a.Hg;
    const bool ub = !LATE && a.tma_b;
    if (threadIdx.x == 0 && (ub || pw_tma)) {
        tma_bar_arm(bar, (uint32_t)((ub ? (FY + 4) * PS * sizeof(T) : 0) + (pw_tma ? 2 * rows * hh * sizeof(T2) : 0)));
        if (ub) tma_load_3d(su_box, &tmu, x0 - 2, y0 - 2, (int)blockIdx.z, bar);
        if (pw_tma) {
            // the pair field as 2 W doubles per row: even half at double 0, odd half at double W
            tma_load_3d(spw, &tmpw, x0 - hle, y0 - a.ha.ht, (int)blockIdx.z, bar);
            tma_load_3d(spw + half, &tmpw, W + x0 - hle, y0 - a.ha.ht, (int)blockIdx.z, bar);
        }
    }
    auto load_u = [&]() {
        if (a.tma_b) return;
        constexpr int UC = FX + 4;
        const int n = (FY + 4) * UC;
        for (int idx = threadIdx.x; idx < n; idx += blockDim.x) {
            const int i = idx / UC, j = idx - i * UC;
            const int yy = y0 - 2 + i, xx = x0 - 2 + j;
            const bool ok = gy0 + yy >= 0 && gy0 + yy < Hg && (a.slab ? (yy >= a.ylo && yy < a.yhi) : (yy >= 0 && yy < H)) &&
                            xx >= 0 && xx < W;
            const uint32_t d = (uint32_t)__cvta_generic_to_shared(su + i * PS + j);
            const T *src = ok ? u + (int64_t)yy * W + xx : u;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(ok ? 8 : 0) : "memory");
        }
    };
    if (!LATE) load_u();
    cp_async_wait_all();
    __syncthreads();
    if (ub || pw_tma) {
        tma_bar_wait(bar);
        __syncthreads();
    }
    const T eps_r2 = a.eps_r2;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ty0 = 4 * warp;
    T2 nd[4][2];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int j = 0; j < 2; ++j) nd[r][j].x = nd[r][j].y = T(0);
    if (LATE) {
        // walk first, then the u tile and the diffusivity over the (p, W) tile
        if (y0 + ty0 < H) adj_walk<T2>(spw + (ty0 + a.ha.ht) * hh + lane, hh, t, nd);
        __syncthreads();
        if (threadIdx.x == 0 && a.tma_b) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            tma_bar_arm(bar2, (uint32_t)((FY + 4) * PS * sizeof(T)));
            tma_load_3d(su_box, &tmu, x0 - 2, y0 - 2, (int)blockIdx.z, bar2);
        }
        load_u();
        cp_async_wait_all();
        __syncthreads();
        if (a.tma_b) {
            tma_bar_wait(bar2);
            __syncthreads();
        }
    }
    if (a.has_d) {
        for (int i = threadIdx.x / 32; i < FY + 2; i += 8) {
            const int yy = y0 - 1 + i;
            const int gyy = gy0 + yy;
            if (gyy < 0 || gyy >= Hg) continue;
            for (int j = threadIdx.x & 31; j < FX + 2; j += 32) {
                const int xx = x0 - 1 + j;
                if (xx < 0 || xx >= W) continue;
                const T *c = su + (i + 1) * PS + (j + 1);
                const T c0 = c[0];
                T q = T(0);
                if (xx + 1 < W) { const T d = c[1] - c0; q += d * d; }
                if (xx > 0) { const T d = c0 - c[-1]; q += d * d; }
                if (gyy + 1 < Hg) { const T d = c[PS] - c0; q += d * d; }
                if (gyy > 0) { const T d = c0 - c[-PS]; q += d * d; }
                sg[i * PS + j] = T(0.5) * frsqrt(T(0.5) * q + eps_r2);
            }
        }
        __syncthreads();
    }
    if (y0 + ty0 >= H) return;
    if (!LATE) adj_walk<T2>(spw + (ty0 + a.ha.ht) * hh + lane, hh, t, nd);
    const T alpha = a.alpha;
    // u rows ty0 + 1 .. ty0 + 6 of the tile (2-pixel halo), columns 2l .. 2l + 5 as three pairs:
    // outputs 2l, 2l + 1 sit at tile columns 2l + 2, 2l + 3
    const T2 *U2 = reinterpret_cast<const T2 *>(su) + lane;            // PS even: rows stay aligned
    const T2 *G2 = reinterpret_cast<const T2 *>(sg) + lane;            // g: columns 2l .. 2l + 3 (1-pixel halo)
    const int xa = x0 + 2 * lane;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int ty = ty0 + k;
        const int y = y0 + ty;
        if (y >= H) break;
        const T2 ua = U2[(ty + 2) * (PS / 2)], ub = U2[(ty + 2) * (PS / 2) + 1], uc = U2[(ty + 2) * (PS / 2) + 2];
        const T2 uu = U2[(ty + 1) * (PS / 2) + 1], ud = U2[(ty + 3) * (PS / 2) + 1];
        T2 ga{}, gb{}, gua{}, gub{}, gda{}, gdb{};
        if (a.has_d) {
            ga = G2[(ty + 1) * (PS / 2)];
            gb = G2[(ty + 1) * (PS / 2) + 1];
            gua = G2[ty * (PS / 2)];
            gub = G2[ty * (PS / 2) + 1];
            gda = G2[(ty + 2) * (PS / 2)];
            gdb = G2[(ty + 2) * (PS / 2) + 1];
        }
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int x = xa + r;
            if (x >= W) continue;
            // centre, left, right, up, down of u; the same of g (k_plane_b_fast's c[..], g[..])
            const T uv = r ? ub.y : ub.x, ul = r ? ub.x : ua.y, ur = r ? uc.x : ub.y;
            const T uup = r ? uu.y : uu.x, udn = r ? ud.y : ud.x;
            T d = T(0);
            if (a.has_d) {
                const T gc = r ? gb.x : ga.y, gl = r ? ga.y : ga.x, gr = r ? gb.y : gb.x;
                const T gup = r ? gub.x : gua.y, gdn = r ? gdb.x : gda.y;
                if (x + 1 < W) d += (gc + gr) * (ur - uv);
                if (x > 0) d -= (gl + gc) * (uv - ul);
                if (gy0 + y + 1 < Hg) d += (gc + gdn) * (udn - uv);
                if (gy0 + y > 0) d -= (gup + gc) * (uv - uup);
            }
            T nm = nd[k][r].x;
            T dn = ROBUST ? nd[k][r].y : T(1);
            if (a.has_d) {
                nm += alpha * dmax_sel(d, T(0));
                dn -= alpha * dmin_sel(d, T(0));
            } else if (!ROBUST) {
                uo[(int64_t)y * W + x] = uv * nm;
                continue;
            }
            dn = dmax_sel(dn, T(kGuard));
            uo[(int64_t)y * W + x] = (uv * nm) * frcp(dn);
        }
    }
}

// ---------------------------------------------------------------------------------- host

// merged columns for k_plane_b_adj (md_plane_fast.h): the union of the dy-runs of tap columns d
// and d - 1 for d = dxmin .. dxmax + 1, zero weights outside each run (and in its interior gaps,
// as build_col_taps); at == nullptr: only check the limits
template <typename T>
bool build_adj_taps(const std::vector<PlaneTap> &taps, int hle, int hh, int rows, AdjTaps<T> *at) {
    std::map<int, std::map<int, double>> by_dx;
    for (const PlaneTap &tp : taps) by_dx[tp.dx][tp.dy] += tp.w;
    int nc = 0, nw = 0;
    if (!by_dx.empty()) {
        const int dmin = by_dx.begin()->first, dmax = by_dx.rbegin()->first + 1;
        for (int d = dmin; d <= dmax; ++d) {
            const auto i0 = by_dx.find(d), i1 = by_dx.find(d - 1);
            if (i0 == by_dx.end() && i1 == by_dx.end()) continue;
            int lo = 1 << 30, hi = -(1 << 30);
            for (const auto &it : {i0, i1})
                if (it != by_dx.end()) {
                    lo = std::min(lo, it->second.begin()->first);
                    hi = std::max(hi, it->second.rbegin()->first);
                }
            const int len = hi - lo + 1;
            if (nc >= kAdjColMax || nw + len > kAdjWeights || len > 0xffff || d + hle < 0) return false;
            if (at) {
                const int e = d + hle;
                const int half = (rows * hh + 7) & ~7;   // k_plane_b_adj's parity halves
                at->c[nc] = make_int2((e & 1) * half + lo * hh + (e >> 1), len | (nw << 16));
                auto wof = [&](std::map<int, std::map<int, double>>::const_iterator it, int dy) {
                    if (it == by_dx.end()) return 0.0;
                    const auto &col = it->second;
                    if (dy < col.begin()->first || dy > col.rbegin()->first) return 0.0;
                    const auto f = col.find(dy);
                    return f == col.end() ? 0.0 : f->second;
                };
                for (int i = 0; i < len; ++i) {
                    at->w[nw + i].x = T(wof(i0, lo + i));
                    at->w[nw + i].y = T(wof(i1, lo + i));
                }
            }
            nw += len;
            ++nc;
        }
    }
    if (at) {
        at->ncol = nc;
        at->hle = hle;
        at->hh = hh;
    }
    return true;
}

// the de-interleaved tile geometry: start column x0 - hle (hle = hl rounded up to even), hh pairs
// per parity half (the tile's FX + hle + hr columns, rounded up to even)
inline void adj_geometry(const PlaneHalo &ha, int *hle, int *hh) {
    *hle = (ha.hl + 1) & ~1;
    *hh = (FX + *hle + ha.hr + 1) / 2;
}
static size_t smem_b_adj(const PlaneHalo &ha, int hh, bool late = false) {
    const size_t pw = (size_t)2 * (((FY + ha.ht + ha.hb) * hh + 7) & ~7) * 16, ug = (size_t)(2 * FY + 6) * PS * 8;
    if (late) return pw < ug ? 0 : pw + 16 + 16;
    return pw + ug + 16 + 8;
}

// + an 8-byte-aligned TMA barrier behind the tile(s); stage B's u tile starts 128-byte aligned
static size_t smem_a(const PlaneHalo &hb, size_t es, int ssa) {
    return (((size_t)(FY + hb.ht + hb.hb) * ssa * es + 7) & ~size_t(7)) + 8;
}
static size_t smem_b(const PlaneHalo &ha, size_t es, int ssb, int mode = 0) {
    const size_t pw = ((size_t)(FY + ha.ht + ha.hb) * ssb * 2 * es + 127) & ~size_t(127);
    const size_t ug = (size_t)(2 * FY + 6) * PS * es;        // u tile + diffusivity
    if (mode == 2) return pw < ug ? 0 : pw + 16 + 16;        // both over the (p, W) tile (0: does not fit)
    // mode 1: the diffusivity over the (p, W) tile (always larger: >= 32 x 64 pairs against 34 x 72)
    return pw + (mode == 1 ? (size_t)(FY + 4) * PS * es : ug) + 16 + 8;
}
// blocks of `smem` bytes that fit one SM (228 KB, 1 KB reserved per block)
static int blocks_per_sm(size_t smem) { return (int)((228 * 1024) / (smem + 1024)); }

bool plane_fast_supported(const PlaneHalo &hb, const PlaneHalo &ha, const std::vector<PlaneTap> &taps_blur,
                          const std::vector<PlaneTap> &taps_adj, int dtype) {
    if (hb.nt > kPlaneMaxTaps || ha.nt > kPlaneMaxTaps) return false;
    if (FX + hb.hl + hb.hr > 32 * PF_CJ || FX + ha.hl + ha.hr > 32 * PF_CJ) return false;   // pf_load column slots
    const size_t es = dtype == 0 ? 8 : 4;
    const int ssa = dtype == 0 ? pf_stride_a<double>(hb) : pf_stride_a<float>(hb);
    const int ssb = dtype == 0 ? pf_stride_b<double>(ha) : pf_stride_b<float>(ha);
    if (smem_a(hb, es, ssa) > 200 * 1024 || smem_b(ha, es, ssb) > 200 * 1024) return false;
    return dtype == 0 ? build_col_taps<double>(taps_blur, ssa, nullptr) && build_col_taps<double>(taps_adj, ssb, nullptr)
                      : build_col_taps<float>(taps_blur, ssa, nullptr) && build_col_taps<float>(taps_adj, ssb, nullptr);
}

template <typename T>
cudaError_t launch_plane_fast(const PlaneFastDesc &d, bool robust, int64_t batch, cudaStream_t st) {
    PlaneFastArgs<T> a{};
    a.u = static_cast<const T *>(d.u);
    a.f = static_cast<const T *>(d.f);
    a.p = static_cast<T *>(d.p);
    a.w = static_cast<T *>(d.w);
    a.u_out = static_cast<T *>(d.u_out);
    a.H = d.H; a.W = d.W; a.periodic = d.periodic;
    a.slab = d.slab; a.gy0 = d.slab ? d.gy0 : 0; a.Hg = d.slab ? d.Hg : d.H;
    a.hb = d.hb; a.ha = d.ha;
    a.ssa = pf_stride_a<T>(d.hb);
    a.ssb = pf_stride_b<T>(d.ha);
    if (!build_col_taps<T>(*d.taps_blur, a.ssa, &a.tb) || !build_col_taps<T>(*d.taps_adj, a.ssb, &a.ta))
        return cudaErrorNotSupported;
    a.alpha = T(d.alpha); a.eps_d2 = T(d.eps_d2); a.eps_r2 = T(d.eps_r2); a.has_d = d.has_d;
    a.lut = d.lut;
    const size_t sa = smem_a(d.hb, sizeof(T), a.ssa);
    size_t sb = smem_b(d.ha, sizeof(T), a.ssb);
#define MD_CHECK_HOST(c) \
    if (!(c)) return cudaErrorInvalidValue
    auto ka = robust ? k_plane_a_fast<T, true> : k_plane_a_fast<T, false>;
    // the shared layout: mode 1 where it fits one more block per SM than mode 0, mode 2 where it
    // fits two more -- the extra barriers cost 13 % (mode 1) on c5's tiles at an equal block count,
    // and mode 2's late u tile about what one extra block gains (c5: 3 vs 2 blocks, 1.8 % slower);
    // the c4 line PSFs run 4 blocks per SM in mode 2 against 2 in mode 0 (2D class -9 %,
    // scripts/plane_mode_ab.sh). MD_PLANE_B_MODE forces a mode (A/B runs).
    int mode = 0;
    {
        static const int m_env = [] { const char *v = std::getenv("MD_PLANE_B_MODE"); return v ? std::atoi(v) : -1; }();
        const int b0 = blocks_per_sm(sb);
        const size_t s1 = smem_b(d.ha, sizeof(T), a.ssb, 1), s2 = smem_b(d.ha, sizeof(T), a.ssb, 2);
        if (m_env >= 0) mode = (m_env == 2 && s2 == 0) ? 0 : (m_env > 2 ? 0 : m_env);
        else if (s2 && blocks_per_sm(s2) >= b0 + 2) mode = 2;
        else if (blocks_per_sm(s1) > b0) mode = 1;
        if (mode) sb = mode == 2 ? s2 : s1;
    }
    auto kb = mode == 2 ? (robust ? k_plane_b_fast<T, true, 2> : k_plane_b_fast<T, false, 2>)
            : mode == 1 ? (robust ? k_plane_b_fast<T, true, 1> : k_plane_b_fast<T, false, 1>)
                        : (robust ? k_plane_b_fast<T, true, 0> : k_plane_b_fast<T, false, 0>);
    cudaError_t e = func_smem_attr((const void *)ka, sa);
    if (e == cudaSuccess) e = func_smem_attr((const void *)kb, sb);
    if (e != cudaSuccess) return e;
    // float64: stage B with adjacent output columns over a de-interleaved (p, W) tile where its
    // merged tap columns fit (MD_PLANE_ADJ=0 at run time: the stride-32 kernel, for A/B runs)
    // float64 stage B with two ADJACENT output columns per thread (k_plane_b_adj, the (p, W) tile
    // de-interleaved by column parity, the u tile loaded over it after the walk) for PSFs wider
    // than tall whose merged columns all take the unrolled walks (<= 8 steps), where it fits at
    // least as many blocks per SM as the stride-32 kernel's layout: 34 % fewer shared wavefronts
    // for 21 % more (zero-weight) FMAs -- c5 / c2 line PSF 3 blocks against 2 (iterations
    // 41.7 -> 38.3 ms), the wide c4 lines 4 blocks each way (2D PSFs 0.3-0.65 us/frame faster); tall
    // PSFs (long columns, which the stride-32 kernel's 4-row walk already shares) keep it
    // (scripts/plane_adjmode_ab.sh). MD_PLANE_ADJ: -1 (default) that pick, 0 off, 2 adjacent
    // columns with separate regions, 3 with the late layout (A/B runs).
    static const int adj_env = [] { const char *v = std::getenv("MD_PLANE_ADJ"); return v ? std::atoi(v) : -1; }();
    AdjTaps<T> at;
    int hle = 0, hh = 0;
    adj_geometry(d.ha, &hle, &hh);
    const size_t sb_sep = smem_b_adj(d.ha, hh, false), sb_late = smem_b_adj(d.ha, hh, true);
    const int blocks_fast = std::min(4, blocks_per_sm(sb));                      // 64 registers
    const int smem_late = sb_late ? blocks_per_sm(sb_late) : 0;
    const bool b4 = smem_late >= 4;                                             // 64 / 80 registers
    const int blocks_adj = std::min(b4 ? 4 : 3, smem_late);
    const bool late = adj_env == 2 ? false : sb_late != 0;
    const bool wide = d.ha.hl + d.ha.hr > d.ha.ht + d.ha.hb;
    const bool want_adj = adj_env == -1 ? (wide && sb_late != 0 && blocks_adj >= blocks_fast) : adj_env >= 2;
    const size_t sb_adj = late ? sb_late : sb_sep;
    bool use_adj = sizeof(T) == 8 && want_adj && (d.W & 1) == 0 && FX + hle + d.ha.hr <= 32 * PF_CJ &&
                   sb_adj <= 200 * 1024 && build_adj_taps<T>(*d.taps_adj, hle, hh, FY + d.ha.ht + d.ha.hb, &at);
    if (use_adj && adj_env == -1)
        for (int c = 0; c < at.ncol; ++c) use_adj = use_adj && (at.c[c].y & 0xffff) <= 8;
    using KB = void (*)(PlaneFastArgs<T>, AdjTaps<T>, CUtensorMap, CUtensorMap);
    KB kb_adj = nullptr;
    if constexpr (sizeof(T) == 8) {
        if (!late) kb_adj = robust ? k_plane_b_adj<T, true, false, false> : k_plane_b_adj<T, false, false, false>;
        else if (b4) kb_adj = robust ? k_plane_b_adj<T, true, true, true> : k_plane_b_adj<T, false, true, true>;
        else kb_adj = robust ? k_plane_b_adj<T, true, true, false> : k_plane_b_adj<T, false, true, false>;
    }
    if (use_adj) {
        e = func_smem_attr((const void *)kb_adj, sb_adj);
        if (e != cudaSuccess) return e;
    }
    const CUtensorMap no_map{};                      // slab launches: per-element tile loads
    a.tma_a = a.tma_b = a.tma_pw = 0;
    a.pwi = d.pw_pairs;
    if (d.slab && d.pw_pairs) return cudaErrorInvalidValue;   // slabs exchange p and W rows separately
    if (d.slab) {
        // stage A over rows [a_begin, a_end) (at most the extended rows [-adj.ht, H + adj.hb)),
        // stage B over own rows [b_begin, b_end): the row-slab driver runs the rows that do not
        // need the neighbours' halo while the halo exchange is in flight (slab.py)
        a.ylo = -d.halo_top;
        a.yhi = d.H + d.halo_bot;
        auto sub = [&](int r0, int r1) {
            PlaneFastArgs<T> s2 = a;
            const int64_t off = (int64_t)r0 * d.W;
            s2.u += off; s2.f += off; s2.p += off; s2.w += off; s2.u_out += off;
            s2.H = r1 - r0; s2.gy0 = d.gy0 + r0;
            s2.ylo = a.ylo - r0; s2.yhi = a.yhi - r0;
            return s2;
        };
        if (d.a_end > d.a_begin) {
            MD_CHECK_HOST(d.a_begin >= -d.ha.ht && d.a_end <= d.H + d.ha.hb);
            ka<<<dim3((d.W + FX - 1) / FX, (d.a_end - d.a_begin + FY - 1) / FY, 1), 256, sa, st>>>(sub(d.a_begin, d.a_end), no_map);
        }
        if (d.b_end > d.b_begin) {
            const dim3 gb((d.W + FX - 1) / FX, (d.b_end - d.b_begin + FY - 1) / FY, 1);
            if (use_adj) kb_adj<<<gb, 256, sb_adj, st>>>(sub(d.b_begin, d.b_end), at, no_map, no_map);
            else kb<<<gb, 256, sb, st>>>(sub(d.b_begin, d.b_end), no_map, no_map);
        }
        return cudaGetLastError();
    }
    const int64_t fsz = (int64_t)d.H * d.W;
    for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
        const int nb = (int)((batch - b0) < 65535 ? (batch - b0) : 65535);
        PlaneFastArgs<T> ab = a;
        ab.u += b0 * fsz; ab.f += b0 * fsz; ab.p += b0 * fsz; ab.w += b0 * fsz; ab.u_out += b0 * fsz;
        const dim3 grid((d.W + FX - 1) / FX, (d.H + FY - 1) / FY, nb);
        // the u tiles by TMA where the maps can be made (16-byte row pitch and box rows)
        CUtensorMap tm_a{}, tm_b{}, tm_pw{};
        static const int tma_mask = [] { const char *e = std::getenv("MD_PLANE_TMA_MASK"); return e ? std::atoi(e) : 7; }();
        ab.tma_a = MD_PLANE_TMA && (tma_mask & 1) && make_tmap_3d(&tm_a, ab.u, sizeof(T), d.W, d.H, nb, a.ssa, FY + d.hb.ht + d.hb.hb);
        ab.tma_b = MD_PLANE_TMA && (tma_mask & 2) && make_tmap_3d(&tm_b, ab.u, sizeof(T), d.W, d.H, nb, PS, FY + 4);
        // interleaved (p, W) pairs as 2W elements per row
        if (use_adj) {
            // stage A writes the pairs parity-split per row; stage B loads each parity half of its
            // tile as one box of the pair field read as 2 W doubles per row
            ab.pw_split = ab.pwi;
            ab.tma_pw = MD_PLANE_TMA && (tma_mask & 4) && ab.pwi &&
                        make_tmap_3d(&tm_pw, ab.p, sizeof(T), 2 * (int64_t)d.W, d.H, nb, 2 * hh, FY + d.ha.ht + d.ha.hb);
            ka<<<grid, 256, sa, st>>>(ab, tm_a);
            kb_adj<<<grid, 256, sb_adj, st>>>(ab, at, tm_b, tm_pw);
            continue;
        }
        ab.tma_pw = MD_PLANE_TMA && (tma_mask & 4) && ab.pwi &&
                    make_tmap_3d(&tm_pw, ab.p, sizeof(T), 2 * (int64_t)d.W, d.H, nb, 2 * a.ssb, FY + d.ha.ht + d.ha.hb);
        ka<<<grid, 256, sa, st>>>(ab, tm_a);
        kb<<<grid, 256, sb, st>>>(ab, tm_b, tm_pw);
    }
    return cudaGetLastError();
}

template cudaError_t launch_plane_fast<double>(const PlaneFastDesc &, bool, int64_t, cudaStream_t);
template cudaError_t launch_plane_fast<float>(const PlaneFastDesc &, bool, int64_t, cudaStream_t);

}  // namespace md
