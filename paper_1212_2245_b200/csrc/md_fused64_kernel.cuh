// md_fused64_kernel.cuh -- the float64 cluster-resident RRRL loop for 1D blur (frames <= 256
// samples per line): all iterations of a frame in ONE launch, the iterate resident in the shared
// memory of a thread-block cluster.
//
// Replaces the iteration loop of DeblurPipeline.run_timed (deconv.py:675-681): _iterate_rrrl
// (deconv.py:512-521) -> _blur_guarded (415-418), _weight_arrays + DivergenceLut.r1 (142-162,
// 114-134), _diffusion_arrays (187-213), _combine (421-446), with the box (conv.py:141-173) or
// dense line-tap convolver, in IEEE float64 throughout (the reference's arithmetic, core.py:3-4).
//
// What differs from the float kernel (md_fused_kernel.cuh), all to fit float64 lines (2.4 KB
// each) at two 8-warp CTAs per SM:
//  * no per-warp p / W line buffers: the adjoint windows of p = W f / b and W are assembled in
//    registers with warp shuffles (a lane's 8 samples plus R from each neighbour lane, the line
//    ends edge-replicated or wrapped), so shared memory holds only the iterate, its halo lines
//    and the diffusivity;
//  * the boundary lines travel to the neighbour CTAs as st.async stores into their shared
//    memory, completing a transaction count on the neighbour's mbarrier (one per halo parity):
//    each CTA waits only for its two neighbours' lines, not for a cluster-wide barrier, and the
//    interior diffusivity is computed while they are in flight;
//  * the divergence table is read as one 16-byte (value, step) pair per pixel (bitwise the
//    reference's T[i] + (T[i+1] - T[i]) t).
//
// Per iteration, per CTA (lines li = warp + NW j):
//   per own line: window of u (smem) -> blur -> guard -> W, p (registers) -> shuffled windows ->
//   adjoint pair -> TV divergence from the stored diffusivity -> u' (registers)
//   __syncthreads; u' -> own lines (+ x-halos); boundary lines -> neighbours (st.async);
//   __syncthreads; interior diffusivity; wait for the neighbours' lines; boundary diffusivity
#pragma once
#include <cooperative_groups.h>

#include <tuple>
#include <cstdlib>

#include "md_fused_kernel.cuh"

namespace md {

// ------------------------------------------------------------------ mbarrier / DSMEM helpers
__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
// the single arrival of a phase plus the bytes it expects from the neighbours
__device__ __forceinline__ void mb_arm(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_wait(uint32_t bar, uint32_t parity) {
    uint32_t done;
#ifdef MD_CHECKED
    long long spins = 0;
#endif
    do {
#ifdef MD_CHECKED
        MD_CHECK(++spins < (1ll << 28));          // a lost arrival / byte count would hang here
#endif
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ uint32_t cluster_map(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
// 16 bytes into a neighbour CTA's shared memory; completes 16 bytes of its mbarrier's count
__device__ __forceinline__ void st_async_f64x2(uint32_t raddr, double x, double y, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(raddr),
                 "d"(x), "d"(y), "r"(rbar)
                 : "memory");
}

// 1D bulk copy (TMA) global -> this CTA's shared memory, completing `bytes` on `bar`
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

// MD_F64_FPOS_TMA=1: the observation line of the next line slot is staged through shared memory
// by the TMA engine (one 2 KB bulk copy per line, per-warp buffer and mbarrier) instead of
// per-lane L2 loads. Measured SLOWER on c1 (iterations 21.8 vs 19.0 ms per 4096 frames): the
// 32 KB of buffers push the CTA's shared memory from 182 to 214 KB, the carveout from 196 to
// 228 KB, and the L1 left for the divergence-table reads from 60 to 28 KB. Off by default.
#ifndef MD_F64_FPOS_TMA
#define MD_F64_FPOS_TMA 0
#endif
constexpr int F64_OBS_LINE = 256;                 // doubles per warp buffer (n <= 256)

// r1 with the (value, step) pair table (md_common.cuh rules, deconv.py:114-134): the table
// interpolation and the linear continuation above `upper`; the direct formula below
// `direct_below` is the caller's (taken per warp, see k_fused_lines64)
// The reference clamps x to `upper` and the position to >= 0 before indexing; both clamps only
// matter where the result is replaced anyway (x > upper: the linear continuation below; x <
// delta < direct_below: the caller's direct formula), so the index is clamped as an integer
// instead (saturating conversion, two integer min/max) -- bitwise the same r1 wherever it is used,
// without the float64 compare-and-select pairs
__device__ __forceinline__ double r1_table64(const double2 *__restrict__ p64, double x) {
    const double pos = (x - kLutDelta) * kLutInvStep;
    int i = __double2int_rz(pos);
    i = min(max(i, 0), kLutCount - 2);
    const double2 e = __ldg(p64 + i);
    double r = e.x + e.y * (pos - (double)i);
    if (x > kLutUpper) r = kLutSlope * x + kLutIntercept;
    return r;
}

// the window [-R, SEG + R) of a lane's 8 samples, the outer 2R taken from the lanes one or two
// segments away (R <= 16; lanes >= nseg idle); clamped line ends replicate the end sample,
// periodic ones wrap
template <int R>
__device__ __forceinline__ void lane_window(const double (&x)[SEG], double (&w)[SEG + 2 * R], int lane, int nseg,
                                            bool periodic) {
    static_assert(R <= 2 * SEG, "neighbour-lane windows need R <= 16");
    auto src = [&](int d) {                       // lane d segments away, wrapped over the line
        int t = lane + d;
        t = t < 0 ? t + nseg : (t >= nseg ? t - nseg : t);
        return t;
    };
    const int l1 = src(-1), r1 = src(1);
    const int l2 = R > SEG ? src(-2) : l1, r2 = R > SEG ? src(2) : r1;
#pragma unroll
    for (int k = 0; k < SEG; ++k) w[R + k] = x[k];
#pragma unroll
    for (int k = 0; k < R; ++k) {
        const int pl = k - R;                     // left position relative to the segment start
        const int el = pl + (pl < -SEG ? 2 * SEG : SEG);
        w[k] = __shfl_sync(0xffffffffu, x[el], pl < -SEG ? l2 : l1);
        const int pr = SEG + k;                   // right position
        const int er = pr - (pr >= 2 * SEG ? 2 * SEG : SEG);
        w[R + SEG + k] = __shfl_sync(0xffffffffu, x[er], pr >= 2 * SEG ? r2 : r1);
    }
    if (!periodic) {
        if constexpr (R <= SEG) {                 // only the end lanes reach past the line
            if (lane == 0)
#pragma unroll
                for (int k = 0; k < R; ++k) w[k] = x[0];
            if (lane == nseg - 1)
#pragma unroll
                for (int k = 0; k < R; ++k) w[R + SEG + k] = x[SEG - 1];
        } else {                                  // two lanes at each end do
            const double first = __shfl_sync(0xffffffffu, x[0], 0);
            const double last = __shfl_sync(0xffffffffu, x[SEG - 1], nseg - 1);
            const int g0 = SEG * lane;            // line position of the segment start
#pragma unroll
            for (int k = 0; k < R; ++k) {
                if (g0 + k - R < 0) w[k] = first;
                if (g0 + SEG + k >= SEG * nseg) w[R + SEG + k] = last;
            }
        }
    }
}

#ifndef MD_F64_SELMAX
#define MD_F64_SELMAX 1            // guards as compare + select (dmax_sel) instead of fmax
#endif
#if MD_F64_SELMAX
#define MD_F64_MAX(a, b) dmax_sel(a, b)
#else
#define MD_F64_MAX(a, b) fmax(a, b)
#endif
#ifndef MD_F64_BLOCKS_PER_SM
#define MD_F64_BLOCKS_PER_SM 1
#endif
// MD_F64_SKIP_SHADOW=1: a warp whose last line slot lies past RL (ragged split: 28-29 lines on
// 16 warps x 2 slots in 9-CTA clusters) skips that slot's arithmetic instead of recomputing line
// RL - 1 (the branch is warp-uniform, so the shuffles inside stay full-warp)
#ifndef MD_F64_GROT
#define MD_F64_GROT g_rot           // measurement knob: (NW - 2) restores the fixed rotation
#endif
#ifndef MD_F64_SKIP_SHADOW
#define MD_F64_SKIP_SHADOW 1
#endif
template <int R, int NW, int LPW, bool ROBUST, int BOXR, bool BOXC>
__global__ void __launch_bounds__(NW * 32, MD_F64_BLOCKS_PER_SM)
k_fused_lines64(FusedKArgs<double, R> a, const double2 *__restrict__ lut64) {
    using T = double;
    constexpr int HW = HaloOf<R>::value;
    constexpr int WIN = SEG + 2 * R;
    constexpr int RLMAX = NW * LPW;                 // line slots per CTA
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T *sm = reinterpret_cast<T *>(smem_raw);
    const int n = a.n, m = a.m;
    const int ls = (xline_len(n, HW) + 1) & ~1;      // even: 16-byte st.async granules
    const int rank = (int)cluster.block_rank();
    const int CL = a.cl;
    const int64_t frame = blockIdx.x / CL;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nseg = n / SEG;
    const int base0 = xaddr(HW);
    // m lines over CL CTAs as evenly as possible (the cluster size is picked on the host for
    // GPC fill, so m / CL need not be an integer): RL = m / CL or one more
    const int lbase = m / CL, lext = m - lbase * CL;
    const int RL = lbase + (rank < lext ? 1 : 0);
    const int gl0 = rank * lbase + (rank < lext ? rank : lext);
    const int64_t fsz = (int64_t)n * m;
    const T *fpos = a.fpos + frame * fsz;

    // shared layout (lines of ls doubles, the same offsets in every CTA of the cluster):
    // own[RLMAX] | halo[parity][top, bottom][2] | g[RLMAX + 2] | mbar[2]
    T *own = sm;
    auto halo = [&](int par, int side) { return sm + (RLMAX + 4 * par + 2 * side) * ls; };
    T *sg = sm + (RLMAX + 8) * ls;
    T *obs_all = sm + (2 * RLMAX + 10) * ls;       // [NW][F64_OBS_LINE] observation lines (TMA)
    uint64_t *mbar = reinterpret_cast<uint64_t *>(obs_all + (MD_F64_FPOS_TMA ? NW * F64_OBS_LINE : 0));
    T *obs = obs_all + warp * F64_OBS_LINE;
    uint64_t *obar = mbar + 2 + warp;             // this warp's observation barrier
    poison_smem(smem_raw);
    MD_CHECK(n % SEG == 0 && nseg <= 32 && RL >= 4 && RL <= RLMAX && CL >= 2 && CL <= 16);
    MD_CHECK((size_t)(2 * RLMAX + 10) * ls * sizeof(T) + 2 * sizeof(uint64_t) <= dyn_smem_bytes());
    auto line_ptr = [&](int l, int par) -> const T * {
        MD_CHECK(l >= -2 && l <= RL + 1 && (par == 0 || par == 1));
        if (l < 0) return halo(par, 0) + (l + 2) * ls;
        if (l >= RL) return halo(par, 1) + (l - RL) * ls;
        return own + l * ls;
    };
    const bool has_top = rank > 0, has_bot = rank < CL - 1;
    const uint32_t line_bytes = (uint32_t)ls * 8u;
    const uint32_t expect = (has_top ? 2u : 0u) * line_bytes + (has_bot ? 2u : 0u) * line_bytes;
    if (threadIdx.x == 0) {
        mb_init(smem_addr(&mbar[0]), 1);
        mb_init(smem_addr(&mbar[1]), 1);
        if (MD_F64_FPOS_TMA)
            for (int w = 0; w < NW; ++w) mb_init(smem_addr(&mbar[2 + w]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        mb_arm(smem_addr(&mbar[0]), expect);
        mb_arm(smem_addr(&mbar[1]), expect);
    }
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    cluster.sync();                                  // all CTAs resident, barriers initialised
    const uint32_t obs_bytes = (uint32_t)n * 8u;
    uint32_t ophase = 0;
    // observation of line slot `li` into this warp's buffer (lane 0)
    auto fetch_obs = [&](int li) {
        if (MD_F64_FPOS_TMA && lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mb_arm(smem_addr(obar), obs_bytes);
            bulk_g2s(smem_addr(obs), fpos + (int64_t)(gl0 + li) * n, obs_bytes, smem_addr(obar));
        }
    };
    if (a.iterations > 0) fetch_obs(min(warp, RL - 1));
    // neighbour targets: my lines 0, 1 -> top neighbour's bottom halo; RL-2, RL-1 -> bottom
    // neighbour's top halo (same parity)
    // parity 0 addresses in the neighbours (parity 1 = + 4 lines, barrier + 8 bytes)
    const uint32_t top_dst = has_top ? cluster_map(smem_addr(halo(0, 1)), rank - 1) : 0u;
    const uint32_t bot_dst = has_bot ? cluster_map(smem_addr(halo(0, 0)), rank + 1) : 0u;
    const uint32_t top_bar = has_top ? cluster_map(smem_addr(&mbar[0]), rank - 1) : 0u;
    const uint32_t bot_bar = has_bot ? cluster_map(smem_addr(&mbar[0]), rank + 1) : 0u;
    // one own line (already in shared memory, x-halos filled) to the neighbour that needs it
    auto push_line = [&](int li, int par) {
        const T *L = own + li * ls;
        uint32_t dst, bar;
        if (li < 2 && has_top) {
            dst = top_dst + (uint32_t)((4 * par + li) * ls) * 8u;
            bar = top_bar + 8u * par;
        } else if (li >= RL - 2 && has_bot) {
            dst = bot_dst + (uint32_t)((4 * par + li - (RL - 2)) * ls) * 8u;
            bar = bot_bar + 8u * par;
        } else {
            return;
        }
        MD_CHECK(li >= 0 && li < RL && (par == 0 || par == 1) && (ls & 1) == 0);
        for (int q = 2 * lane; q < ls; q += 64) st_async_f64x2(dst + (uint32_t)q * 8u, L[q], L[q + 1], bar);
    };

    // ---- load u0 (own lines), fill x-halos, push the boundary lines (parity 0)
    {
        const T *src = a.u0 + frame * fsz + (int64_t)gl0 * n;
        for (int li = warp; li < RL; li += NW) {
            T *L = own + li * ls;
            for (int j = lane; j < n; j += 32) L[xaddr(HW + j)] = src[(int64_t)li * n + j];
            __syncwarp();
            fu_fill_halo<T>(L, n, HW, a.periodic, lane);
            __syncwarp();
            push_line(li, 0);
        }
    }

    const T eps_r2 = a.eps_r2, eps_d2 = a.eps_d2;
    constexpr bool FOLD = BOXR > 0 && !BOXC;
    const T al = FOLD ? a.alpha_w : a.alpha, gd = FOLD ? a.guard_w : T(kGuard), one = FOLD ? a.one_w : T(1);
    // diffusivity g on logical lines l in [lb, le] (deconv.py:191-203)
    auto g_lines = [&](int lb, int le, int par, int wl) {
        if (!a.has_d) return;
        for (int l = lb + wl; l <= le; l += NW) {
            const int gl = gl0 + l;
            if (gl < 0 || gl >= m) continue;
            // Neumann at the frame's first / last line: the missing neighbour aliases the line
            // itself, so its difference is exactly zero (no per-pixel selects)
            const T *row = line_ptr(l, par);
            const T *up = gl > 0 ? line_ptr(l - 1, par) : row, *dn = gl + 1 < m ? line_ptr(l + 1, par) : row;
            for (int s = lane; s < nseg; s += 32) {
                const int off = base0 + 9 * s;
                T x[SEG + 2];
#pragma unroll
                for (int k = -1; k <= SEG; ++k) x[k + 1] = row[off + koff(k)];
                MD_CHECK(l >= -1 && l <= RL);
                T *G = sg + (l + 1) * ls + off;
#pragma unroll
                for (int r = 0; r < SEG; ++r) {
                    T dxr = x[r + 2] - x[r + 1];
                    T dxl = x[r + 1] - x[r];
                    if (r == SEG - 1 && s == nseg - 1) dxr = T(0);
                    if (r == 0 && s == 0) dxl = T(0);
                    const T dyd = dn[off + koff(r)] - x[r + 1], dyu = x[r + 1] - up[off + koff(r)];
                    const T q = dxr * dxr + dxl * dxl + dyd * dyd + dyu * dyu;
                    G[koff(r)] = T(0.5) * frsqrt(T(0.5) * q + eps_r2);
                }
            }
        }
    };
    // wait for the neighbours' lines of parity `par` (phase `use` of that barrier), re-arm it,
    // then the diffusivity of the halo-dependent lines
    // interior diffusivity lines 1 .. RL-2 dealt so that warps 0-3, which take the four
    // halo-dependent lines after the neighbours' wait, are among the warps with one interior line:
    // NW - min(4, ones) with `ones` warps holding a single interior line (RL = 28 / 29 in 9-CTA
    // clusters: 6 / 5 such warps; RL = 32: 2 -- the former fixed NW - 2)
    const int g_ones = 2 * NW - (RL - 2);
    const int g_rot = NW - (g_ones < 4 ? (g_ones > 0 ? g_ones : 0) : 4);
    auto publish_and_g = [&](int par, int use) {
        __syncthreads();
        g_lines(1, RL - 2, par, (warp + MD_F64_GROT) % NW);
        if (warp < 4) {
            mb_wait(smem_addr(&mbar[par]), (uint32_t)(use & 1));
            if (threadIdx.x == 0) mb_arm(smem_addr(&mbar[par]), expect);
            g_lines(warp < 2 ? -1 : RL - 1, warp < 2 ? 0 : RL, par, warp & 1);
        }
        __syncthreads();
    };
    publish_and_g(0, 0);
    for (int it = 0; it < a.iterations; ++it) {
        const int par = it & 1;
        const bool last = it == a.iterations - 1;
        T unew[LPW][SEG];
#pragma unroll
        for (int j = 0; j < LPW; ++j) {
            // slots past RL (ragged line split) shadow line RL - 1 and store nothing: the loop
            // stays convergent, so the shuffles need no per-iteration reconvergence
            // (MD_F64_SKIP_SHADOW: the whole warp skips such a slot -- the test is warp-uniform)
            if (MD_F64_SKIP_SHADOW && j > 0 && warp + NW * j >= RL) continue;
            const int li = min(warp + NW * j, RL - 1);
            const int gl = gl0 + li;
            const bool up_ok = gl > 0, dn_ok = gl + 1 < m;
            const T *U = own + li * ls;
            const int s = lane < nseg ? lane : nseg - 1;     // idle lanes shadow the last segment
            const int off = base0 + 9 * s;
            const int ln = j + 1 < LPW ? min(warp + NW * (j + 1), RL - 1) : min(warp, RL - 1);
            T fv[SEG];
            if (MD_F64_FPOS_TMA) {
                mb_wait(smem_addr(obar), ophase);
                ophase ^= 1u;
                const double2 *f2 = reinterpret_cast<const double2 *>(obs + SEG * s);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const double2 x = f2[i];
                    fv[2 * i] = x.x;
                    fv[2 * i + 1] = x.y;
                }
                __syncwarp();
                if (!(last && j == LPW - 1)) fetch_obs(ln);   // the next slot's line, in flight meanwhile
            } else {
                const T *F = fpos + (int64_t)gl * n;
                asm volatile("prefetch.global.L1 [%0];" ::"l"(fpos + (int64_t)(gl0 + ln) * n + SEG * s));
                const double2 *f2 = reinterpret_cast<const double2 *>(F + SEG * s);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const double2 x = __ldg(f2 + i);
                    fv[2 * i] = x.x;
                    fv[2 * i + 1] = x.y;
                }
            }
            T pv[SEG], wv[SEG];
            {
                T v[WIN];
#pragma unroll
                for (int k = -R; k < SEG + R; ++k) v[k + R] = U[off + koff(k)];
                T bl[SEG];
                conv_window<T, R, BOXR, BOXC>(v, a.wb, a.box_wi, a.box_cb, bl);
#pragma unroll
                for (int r = 0; r < SEG; ++r) bl[r] = MD_F64_MAX(bl[r], T(kGuard));   // b
                if (a.floor_f) {
                    // the raw observation: max(f, floor) as the Wiener epilogue forms it (no fpos
                    // field) -- here, after the blur, so the loads' latency hides behind it
#pragma unroll
                    for (int r = 0; r < SEG; ++r) fv[r] = fv[r] > a.floor ? fv[r] : a.floor;
                }
                if (ROBUST) {
                    // r1(b / fpos) for the lane's 8 pixels: all 8 table pairs requested before any
                    // is used (no branch between them), the rare direct-log branch (x < 1/2) taken
                    // once per warp and only when some lane needs it
                    T xr[SEG], r1v[SEG];
                    bool need_log = false;
#pragma unroll
                    for (int r = 0; r < SEG; ++r) {
                        xr[r] = bl[r] * frcp(fv[r]);
                        need_log |= xr[r] < kLutDirectBelow;
                    }
#pragma unroll
                    for (int r = 0; r < SEG; ++r) r1v[r] = r1_table64(lut64, xr[r]);
                    if (__any_sync(0xffffffffu, need_log)) {
#pragma unroll
                        for (int r = 0; r < SEG; ++r)
                            if (xr[r] < kLutDirectBelow) r1v[r] = xr[r] - 1.0 - log(xr[r]);
                    }
#pragma unroll
                    for (int r = 0; r < SEG; ++r) {
                        const T w = T(0.5) * frsqrt(r1v[r] * fv[r] + eps_d2);
                        wv[r] = w;
                        pv[r] = w * (fv[r] * frcp(bl[r]));
                    }
                } else {
#pragma unroll
                    for (int r = 0; r < SEG; ++r) pv[r] = fv[r] * frcp(bl[r]);
                }
            }
            T num[SEG], den[SEG];
            {
                T v[WIN];
                lane_window<R>(pv, v, lane, nseg, a.periodic);
                conv_window<T, R, BOXR, BOXC, !FOLD>(v, a.wa, a.box_wi, a.box_ca, num);
            }
            if (ROBUST) {
                T v[WIN];
                lane_window<R>(wv, v, lane, nseg, a.periodic);
                conv_window<T, R, BOXR, BOXC, !FOLD>(v, a.wa, a.box_wi, a.box_ca, den);
            }
            T ux[SEG + 2];
#pragma unroll
            for (int k = -1; k <= SEG; ++k) ux[k + 1] = U[off + koff(k)];
            if (a.has_d) {
                // Neumann at the frame's first / last line by aliasing (see g_lines): the vertical
                // flux to a missing neighbour is (g + g) (u - u) = 0 exactly
                const T *G = sg + (li + 1) * ls + off;
                const T *Gu = up_ok ? G - ls : G, *Gd = dn_ok ? G + ls : G;
                const T *Uu = up_ok ? line_ptr(li - 1, par) + off : U + off;
                const T *Ud = dn_ok ? line_ptr(li + 1, par) + off : U + off;
                T gx[SEG + 2];
#pragma unroll
                for (int k = -1; k <= SEG; ++k) gx[k + 1] = G[koff(k)];
#pragma unroll
                for (int r = 0; r < SEG; ++r) {
                    const T u = ux[r + 1], gc = gx[r + 1];
                    T fr = (gc + gx[r + 2]) * (ux[r + 2] - u);
                    T fl = (gx[r] + gc) * (u - ux[r]);
                    if (r == SEG - 1 && s == nseg - 1) fr = T(0);
                    if (r == 0 && s == 0) fl = T(0);
                    T d = fr - fl;
                    d += (gc + Gd[koff(r)]) * (Ud[koff(r)] - u);
                    d -= (Gu[koff(r)] + gc) * (u - Uu[koff(r)]);
                    const T dp = MD_F64_MAX(d, T(0));    // max(D, 0); D - max(D, 0) = min(D, 0) exactly
                    const T nm = num[r] + al * dp;
                    const T neg = al * (d - dp);
                    T dn = (ROBUST ? den[r] : one) - neg;
                    dn = MD_F64_MAX(dn, gd);
                    unew[j][r] = (u * nm) * frcp(dn);
                }
            } else {
#pragma unroll
                for (int r = 0; r < SEG; ++r) {
                    if (ROBUST) {
                        const T dn = MD_F64_MAX(den[r], gd);
                        unew[j][r] = (ux[r + 1] * num[r]) * frcp(dn);
                    } else {
                        unew[j][r] = ux[r + 1] * (FOLD ? num[r] * a.box_wi : num[r]);
                    }
                }
            }
        }
        __syncthreads();
        if (last) {
            T *dst = a.out + frame * fsz;
#pragma unroll
            for (int j = 0; j < LPW; ++j) {
                const int li = warp + NW * j;
                const int gl = gl0 + li;
                if (lane >= nseg || li >= RL) continue;
                if (!a.out_vert) {
                    double2 *o2 = reinterpret_cast<double2 *>(dst + (int64_t)gl * n + SEG * lane);
#pragma unroll
                    for (int i = 0; i < 4; ++i) o2[i] = make_double2(unew[j][2 * i], unew[j][2 * i + 1]);
                } else {
                    T *L = own + li * ls + base0 + 9 * lane;
#pragma unroll
                    for (int r = 0; r < SEG; ++r) L[koff(r)] = unew[j][r];
                }
            }
            if (a.out_vert) {
                __syncthreads();
                for (int idx = threadIdx.x; idx < RL * n; idx += blockDim.x) {
                    const int row = idx / RL, li = idx - row * RL;
                    dst[(int64_t)row * m + gl0 + li] = own[li * ls + xaddr(HW + row)];
                }
            }
            break;
        }
        // ---- u' -> own lines + x-halos; boundary lines -> the neighbours' halo[par ^ 1]
        const int npar = par ^ 1;
#pragma unroll
        for (int j = 0; j < LPW; ++j) {
            const int li = warp + NW * j;
            if (li >= RL) continue;
            T *L = own + li * ls;
            if (lane < nseg) {
                T *P = L + base0 + 9 * lane;
#pragma unroll
                for (int r = 0; r < SEG; ++r) P[koff(r)] = unew[j][r];
            }
            __syncwarp();
            fu_fill_halo<T>(L, n, HW, a.periodic, lane);
            __syncwarp();
            push_line(li, npar);
        }
        // use index of barrier npar: u^(it+1) is its ((it + 1) >> 1)-th completion
        publish_and_g(npar, (it + 1) >> 1);
    }
}

template <int R, int NW, int LPW>
size_t fused64_smem(int n) {
    constexpr int HW = HaloOf<R>::value;
    const int ls = (xline_len(n, HW) + 1) & ~1;
    return (size_t)(2 * NW * LPW + 10) * ls * sizeof(double) +
           (MD_F64_FPOS_TMA ? (size_t)NW * F64_OBS_LINE * sizeof(double) : 0) + (2 + NW) * sizeof(uint64_t);
}

// host: the cluster size for m lines -- every CTA holds at most `rlmax` lines and at least 4, one
// CTA per SM. Clusters are placed whole inside a GPC, so the resident count does not scale with
// 1 / size (B200, one CTA per SM: 8-CTA clusters 15 resident = 120 SMs, 9-CTA 15 = 135 SMs,
// 16-CTA 7 = 112 SMs; scripts/probes/cluster_geom.cu). Among the admissible sizes, the most
// frames in flight per line round (each warp's lines run in turn); ties to the smaller cluster.
// Cached per (kernel, smem, m, device).
inline int pick_cluster(const void *kern, size_t smem, int threads, int m, int rlmax, int *resident) {
    static std::mutex mu;
    static std::map<std::tuple<const void *, size_t, int, int>, std::pair<int, int>> memo;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    std::lock_guard<std::mutex> lock(mu);
    const auto key = std::make_tuple(kern, smem, m, dev);
    auto it = memo.find(key);
    if (it == memo.end()) {
        int best = 0, best_n = 0, best_rounds = 1;
        // MD_F64_CLUSTER=k (measurement knob): only cluster size k is considered
        const char *force = std::getenv("MD_F64_CLUSTER");
        const int fcl = force ? std::atoi(force) : 0;
        for (int cl = std::max(2, (m + rlmax - 1) / rlmax); cl <= 16 && m / cl >= 4; ++cl) {
            if (fcl > 0 && cl != fcl) continue;
            cudaLaunchConfig_t q = {};
            q.gridDim = dim3((unsigned)cl, 1, 1);
            q.blockDim = dim3((unsigned)threads, 1, 1);
            q.dynamicSmemBytes = smem;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = cl;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            q.attrs = at;
            q.numAttrs = 1;
            int n = 0;
            if (cudaOccupancyMaxActiveClusters(&n, kern, &q) != cudaSuccess) {
                cudaGetLastError();
                continue;
            }
            // throughput ~ frames in flight / line rounds per frame (a warp's lines run in turn);
            // on a tie the size that keeps more SMs busy (c1: 9 x 15 = 135 SMs at 29 lines per
            // CTA ran 1.7 % faster than 8 x 15 = 120 at 32 lines, scripts/r2_cl_ab.sh)
            const int nw = threads / 32;
            const int rounds = ((m + cl - 1) / cl + nw - 1) / nw;
            const int64_t lhs = (int64_t)n * best_rounds, rhs = (int64_t)best_n * rounds;
            if (best == 0 || lhs > rhs || (lhs == rhs && n * cl > best_n * best)) {
                best = cl; best_n = n; best_rounds = rounds;
            }
        }
        it = memo.emplace(key, std::make_pair(best, best_n)).first;
    }
    if (resident) *resident = it->second.second;
    return it->second.first;
}

template <int R, int NW, int LPW>
cudaError_t launch_fused64_t(void (*kern)(FusedKArgs<double, R>, const double2 *), const FusedKArgs<double, R> &a0,
                             const double2 *lut64, int64_t batch, cudaStream_t st, int *query_geom = nullptr) {
    const size_t smem = fused64_smem<R, NW, LPW>(a0.n);
    {
        const cudaError_t e = func_smem_attr((const void *)kern, smem, true);
        if (e != cudaSuccess) return e;
    }
    FusedKArgs<double, R> a = a0;
    int resident = 0;
    a.cl = pick_cluster((const void *)kern, smem, NW * 32, a.m, NW * LPW, &resident);
    if (a.cl == 0) return cudaErrorNotSupported;
    if (a.query) {
        *a.query = resident;
        if (query_geom) {
            query_geom[0] = a.cl;
            int per_sm = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NW * 32, smem);
            query_geom[1] = per_sm;
        }
        return cudaSuccess;
    }
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = a.cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    const int64_t fsz = (int64_t)a.n * a.m;
    const int64_t maxf = (int64_t)(0x7fffffff / a.cl);
    for (int64_t b0 = 0; b0 < batch; b0 += maxf) {
        const int64_t nb = std::min<int64_t>(maxf, batch - b0);
        FusedKArgs<double, R> ab = a;
        ab.u0 += b0 * fsz;
        ab.fpos += b0 * fsz;
        ab.out += b0 * fsz;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(nb * a.cl), 1, 1);
        cfg.blockDim = dim3(NW * 32, 1, 1);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ab, lut64);
        if (e != cudaSuccess) return e;
    }
    return cudaGetLastError();
}

// geometry of the float64 kernel: 16 warps x 2 line slots (up to 32 lines per CTA, one CTA per
// SM), the cluster size picked per line count (pick_cluster). Measured (c1, 4096 frames):
// 8 warps x 2 lines at two CTAs per SM in 16-CTA clusters (14 resident = 112 SMs) 20.3 ms of
// iterations; 16 x 2 in 8-CTA clusters (15 = 120 SMs) 18.7 ms
#ifndef MD_F64_NW
#define MD_F64_NW 16
#endif
constexpr int F64_NW = MD_F64_NW;
#ifndef MD_F64_LPW
#define MD_F64_LPW 2
#endif
constexpr int F64_LPW = MD_F64_LPW;

template <int RR>
cudaError_t launch_fused64_box_r(const FusedLinesArgs &d, int64_t batch, cudaStream_t st) {
    FusedKArgs<double, RR> a{};
    a.u0 = static_cast<const double *>(d.u_in);
    a.fpos = static_cast<const double *>(d.fpos);
    a.out = static_cast<double *>(d.u_out);
    a.query = d.query;
    a.n = d.n; a.m = d.m; a.iterations = d.iterations; a.out_vert = d.out_vert;
    a.periodic = d.blur.periodic;
    a.cl = 0;                                    // picked at launch (pick_cluster)
    a.alpha = d.alpha; a.eps_d2 = d.eps_d2; a.eps_r2 = d.eps_r2; a.has_d = d.has_d;
    a.lut = d.lut;
    a.floor = d.floor; a.floor_f = d.floor_f;
    a.box_wi = d.blur.wi;
    a.alpha_w = d.alpha / d.blur.wi; a.guard_w = kGuard / d.blur.wi; a.one_w = 1.0 / d.blur.wi;
    if (!box_corrections<double, RR>(d.blur, d.blur.wi, a.box_cb) || !box_corrections<double, RR>(d.adj, d.blur.wi, a.box_ca))
        return cudaErrorNotSupported;
    bool corr = false;
    for (int i = 0; i < 4; ++i) corr = corr || a.box_cb[i] != 0.0 || a.box_ca[i] != 0.0;
    return launch_fused64_t<RR, F64_NW, F64_LPW>(corr ? k_fused_lines64<RR, F64_NW, F64_LPW, true, RR, true>
                                                      : k_fused_lines64<RR, F64_NW, F64_LPW, true, RR, false>,
                                                 a, d.lut.p64, batch, st, d.query_geom);
}

}  // namespace md
