// md_fused_kernel.cuh -- all RRRL iterations of a frame in ONE launch, the iterate resident in the
// distributed shared memory of a thread-block cluster (1D blur scenarios, small frames).
//
// Replaces the iteration loop of DeblurPipeline.run_timed (deconv.py:675-681) with
// _iterate_rrrl and its callees (deconv.py:142-213, 415-446, 512-521) for box / 1D kernels.
//
// Geometry: one cluster of CL CTAs per frame; CTA `rank` owns RL = 8 * LPW consecutive
// lines (line-major layout, lines along the blur axis). The blur and its adjoint act along
// a line (warp-local, register windows, md_linefast.cuh); only the TV stencil couples
// lines, so per iteration a CTA needs its neighbours' two boundary lines. Those are pushed
// into the neighbours' shared memory (DSMEM stores, double-buffered by iteration parity)
// and one cluster barrier per iteration publishes them. The observation is re-read from L2
// (line-major, coalesced) each iteration; HBM sees u0/fpos in and u out only.
//
// Per iteration, per CTA:
//   g on lines -1..RL (needs lines -2..RL+1)         | barrier
//   per own line (warp): blur -> W, p (warp buffer) -> adjoint pair -> D -> u' in registers
//   barrier; u' -> own smem lines; boundary lines -> neighbours' halo[parity^1]; cluster barrier
#pragma once
#include <cooperative_groups.h>

#include "md_fused.h"
#include "md_lines_fast.h"
#include "md_linefast.cuh"

namespace cg = cooperative_groups;

namespace md {

constexpr int FU_WARPS = 8;

template <typename T, int R> struct FusedKArgs {
    const T *u0;        // line-major clamped Wiener output [frames][m][n]
    const T *fpos;      // line-major max(f, floor)
    T *out;             // native layout result
    int *query;         // host: non-null = report the resident cluster count instead of launching
    int n, m, iterations, out_vert, periodic, cl;
    DenseTaps<T, R> wb, wa;
    T alpha, eps_d2, eps_r2;
    int has_d;
    LutView lut;
    T box_wi;           // box specialisation: interior weight
    T alpha_w, guard_w, one_w;   // alpha, the division guard and 1 divided by box_wi
    T box_cb[4], box_ca[4];   // weight corrections at k = -R, -R+1, R-1, R (blur, adjoint)
    T floor;            // floor_f: fpos holds the raw observation, floored on load (float64 kernel)
    int floor_f;
};

__device__ __forceinline__ int fu_wrap(int j, int n, int periodic) {
    // halos never exceed the extent, so one conditional wrap suffices (no integer modulo)
    if (periodic) return j < 0 ? j + n : (j >= n ? j - n : j);
    return j < 0 ? 0 : (j >= n ? n - 1 : j);
}

template <typename T>
__device__ __forceinline__ void fu_fill_halo(T *line, int n, int hw, int periodic, int lane) {
    for (int q = lane; q < 2 * hw; q += 32) {
        const int e = q < hw ? q : n + q;
        line[xaddr(e)] = line[xaddr(hw + fu_wrap(e - hw, n, periodic))];
    }
}

template <typename T, int R, int LPW, bool ROBUST, int BOXR, bool BOXC>
__global__ void __launch_bounds__(256, sizeof(T) == 4 ? (LPW == 2 && R <= 8 ? 3 : 2) : 1)
k_fused_lines(FusedKArgs<T, R> a) {
    constexpr int HW = HaloOf<R>::value;
    constexpr int WIN = SEG + 2 * R;
    constexpr int RL = FU_WARPS * LPW;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T *sm = reinterpret_cast<T *>(smem_raw);
    const int n = a.n, m = a.m;
    const int ls = xline_len(n, HW);
    const int rank = (int)cluster.block_rank();
    const int CL = a.cl;
    const int64_t frame = blockIdx.x / CL;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nseg = n / SEG;
    const int base0 = xaddr(HW);
    const int gl0 = rank * RL;                       // first global line owned
    const int64_t fsz = (int64_t)n * m;
    const T *fpos = a.fpos + frame * fsz;

    // shared layout (in lines of `ls` elements)
    T *own = sm;                                     // RL lines
    auto halo_top = [&](int par) { return sm + (RL + 2 * par) * ls; };
    auto halo_bot = [&](int par) { return sm + (RL + 4 + 2 * par) * ls; };
    T *sg = sm + (RL + 8) * ls;                      // RL+2 lines: logical -1..RL
    T *wp = sm + (2 * RL + 10 + 2 * warp) * ls;      // warp buffers: p, W
    T *ww = wp + ls;
    poison_smem(smem_raw);
    MD_CHECK(m == RL * CL && n % SEG == 0 && n / SEG <= 32);
    MD_CHECK((size_t)(2 * RL + 10 + 2 * FU_WARPS) * ls * sizeof(T) <= dyn_smem_bytes());
    auto line_ptr = [&](int l, int par) -> T * {
        MD_CHECK(l >= -2 && l <= RL + 1 && (par == 0 || par == 1));
        if (l < 0) return halo_top(par) + (l + 2) * ls;
        if (l >= RL) return halo_bot(par) + (l - RL) * ls;
        return own + l * ls;
    };

    // the next chunk's Wiener step is a programmatic dependent launch (md_capi.cu,
    // run_lines_pipelined): it starts once every CTA of this grid has started, i.e. during the
    // last wave, on the SMs the wave leaves free
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    cluster.sync();                                  // all CTAs resident before DSMEM traffic
    T *nb_top = rank > 0 ? cluster.map_shared_rank(sm, rank - 1) : nullptr;
    T *nb_bot = rank < CL - 1 ? cluster.map_shared_rank(sm, rank + 1) : nullptr;

    // ---- load u0 (own lines), fill x-halos, push boundary lines to the neighbours (parity 0)
    {
        const T *src = a.u0 + frame * fsz + (int64_t)gl0 * n;
        for (int li = warp; li < RL; li += FU_WARPS) {
            T *L = own + li * ls;
            for (int j = lane; j < n; j += 32) L[xaddr(HW + j)] = src[(int64_t)li * n + j];
            __syncwarp();
            fu_fill_halo<T>(L, n, HW, a.periodic, lane);
            __syncwarp();
            if (li < 2 && nb_top)
                for (int q = lane; q < ls; q += 32) (nb_top + (RL + 4 + li) * ls)[q] = L[q];
            if (li >= RL - 2 && nb_bot)   // neighbour's top halo (parity 0), logical line li - RL
                for (int q = lane; q < ls; q += 32) (nb_bot + (RL + (li - RL) + 2) * ls)[q] = L[q];
        }
    }

    const T eps_r2 = a.eps_r2, eps_d2 = a.eps_d2;
    // plain integer box: the adjoint window sums stay unscaled and alpha, the guard and the
    // unit denominator carry 1/wi instead -- u (wi S_p + a D+) / (wi S_W - a D-) =
    // u (S_p + (a/wi) D+) / (S_W - (a/wi) D-): two multiplies per pixel fewer
    constexpr bool FOLD = BOXR > 0 && !BOXC;
    const T al = FOLD ? a.alpha_w : a.alpha, gd = FOLD ? a.guard_w : T(kGuard), one = FOLD ? a.one_w : T(1);
    // diffusivity g on logical lines l in [lb, le] (deconv.py:191-203); lines whose stencil
    // touches a halo (l <= 0 or l >= RL-1) need the neighbours' rows of parity `par`
    auto g_lines = [&](int lb, int le, int par, int wl) {
        if (!a.has_d) return;
        for (int l = lb + wl; l <= le; l += FU_WARPS) {
            const int gl = gl0 + l;
            if (gl < 0 || gl >= m) continue;
            const bool up_ok = gl > 0, dn_ok = gl + 1 < m;
            const T *row = line_ptr(l, par), *up = line_ptr(l - 1, par), *dn = line_ptr(l + 1, par);
            for (int s = lane; s < nseg; s += 32) {
                const int off = base0 + 9 * s;
                T x[SEG + 2];
#pragma unroll
                for (int k = -1; k <= SEG; ++k) x[k + 1] = row[off + koff(k)];
                T *G = sg + (l + 1) * ls + off;
#pragma unroll
                for (int r = 0; r < SEG; ++r) {
                    T dxr = x[r + 2] - x[r + 1];
                    T dxl = x[r + 1] - x[r];
                    if (r == SEG - 1 && s == nseg - 1) dxr = T(0);
                    if (r == 0 && s == 0) dxl = T(0);
                    const T yd = dn_ok ? dn[off + koff(r)] : x[r + 1];
                    const T yu = up_ok ? up[off + koff(r)] : x[r + 1];
                    const T dyd = yd - x[r + 1], dyu = x[r + 1] - yu;
                    const T q = dxr * dxr + dxl * dxl + dyd * dyd + dyu * dyu;
                    // float: 0.5 / sqrt(q/2 + eps^2) as 1 / sqrt(2 q + 4 eps^2) (no scaling multiply)
                    G[koff(r)] = sizeof(T) == 4 ? frsqrt(T(2) * q + T(4) * eps_r2) : T(0.5) * frsqrt(T(0.5) * q + eps_r2);
                }
            }
        }
    };
    // split cluster barrier: release my DSMEM stores, compute the interior diffusivity (own
    // lines only) while the neighbours catch up, then acquire and finish the boundary lines
    auto publish_and_g = [&](int par) {
        __syncthreads();
        asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
        // interior lines dealt from warp 2 on (warps 0 and 1 get one line fewer when RL - 2 is
        // not a multiple of 8); the four halo-dependent lines go one each to warps 0..3, so
        // the critical path after the wait is a single line
#ifndef MD_FU_GOLDBAL
        g_lines(1, RL - 2, par, (warp + FU_WARPS - 2) % FU_WARPS);
        asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
        if (warp < 4) g_lines(warp < 2 ? -1 : RL - 1, warp < 2 ? 0 : RL, par, warp & 1);
#else
        g_lines(1, RL - 2, par, warp);
        asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
        g_lines(-1, 0, par, warp);
        g_lines(RL - 1, RL, par, warp);
#endif
        __syncthreads();
    };
    publish_and_g(0);
    for (int it = 0; it < a.iterations; ++it) {
        const int par = it & 1;
        const bool last = it == a.iterations - 1;
        // ---- per own line: blur -> W, p -> adjoint pair -> D -> update (registers)
        T unew[LPW][SEG];
#pragma unroll
        for (int j = 0; j < LPW; ++j) {
            const int li = warp + FU_WARPS * j;
            const int gl = gl0 + li;
            const bool up_ok = gl > 0, dn_ok = gl + 1 < m;
            const T *U = own + li * ls;
            const T *F = fpos + (int64_t)gl * n;
            // nseg <= 32 (n <= 256): one segment per lane
            const int s = lane;
            const bool act = s < nseg;
            const int off = base0 + 9 * s;
            if (act) {
                // the observation of this warp's next line (next iteration's first line after the
                // last) into L1 now, so its load below hits L1 instead of waiting on L2
                const int ln = j + 1 < LPW ? li + FU_WARPS : warp;
                asm volatile("prefetch.global.L1 [%0];" ::"l"(fpos + (int64_t)(gl0 + ln) * n + SEG * s));
                T fv[SEG];
                if (sizeof(T) == 4) {
                    const float4 *f4 = reinterpret_cast<const float4 *>(F + SEG * s);
                    const float4 x0 = __ldg(f4), x1 = __ldg(f4 + 1);
                    fv[0] = x0.x; fv[1] = x0.y; fv[2] = x0.z; fv[3] = x0.w;
                    fv[4] = x1.x; fv[5] = x1.y; fv[6] = x1.z; fv[7] = x1.w;
                } else {
                    const double2 *f2 = reinterpret_cast<const double2 *>(F + SEG * s);
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const double2 x = __ldg(f2 + i);
                        fv[2 * i] = (T)x.x;
                        fv[2 * i + 1] = (T)x.y;
                    }
                }
                T v[WIN];
#pragma unroll
                for (int k = -R; k < SEG + R; ++k) v[k + R] = U[off + koff(k)];
                T bl[SEG];
                conv_window<T, R, BOXR, BOXC>(v, a.wb, a.box_wi, a.box_cb, bl);
#pragma unroll
                for (int r = 0; r < SEG; ++r) {
                    const T b = bl[r] > T(kGuard) ? bl[r] : T(kGuard);
                    const T fp = fv[r];
                    const T ratio = fp * frcp(b);
                    if (ROBUST) {
                        const T xr = b * frcp(fp);
                        const T w = T(0.5) * frsqrt(r1_fast<T>(a.lut, xr) * fp + eps_d2);
                        ww[off + koff(r)] = w;
                        wp[off + koff(r)] = w * ratio;
                    } else {
                        wp[off + koff(r)] = ratio;
                    }
                }
            }
            __syncwarp();
            fu_fill_halo<T>(wp, n, HW, a.periodic, lane);
            if (ROBUST) fu_fill_halo<T>(ww, n, HW, a.periodic, lane);
            __syncwarp();
            if (act) {
                T num[SEG], den[SEG];
                {
                    T v[WIN];
#pragma unroll
                    for (int k = -R; k < SEG + R; ++k) v[k + R] = wp[off + koff(k)];
                    conv_window<T, R, BOXR, BOXC, !FOLD>(v, a.wa, a.box_wi, a.box_ca, num);
                }
                if (ROBUST) {
                    T v[WIN];
#pragma unroll
                    for (int k = -R; k < SEG + R; ++k) v[k + R] = ww[off + koff(k)];
                    conv_window<T, R, BOXR, BOXC, !FOLD>(v, a.wa, a.box_wi, a.box_ca, den);
                }
                T ux[SEG + 2];
#pragma unroll
                for (int k = -1; k <= SEG; ++k) ux[k + 1] = U[off + koff(k)];
                if (a.has_d) {
                    const T *G = sg + (li + 1) * ls + off;
                    const T *Gu = G - ls, *Gd = G + ls;
                    const T *Uu = line_ptr(li - 1, par) + off, *Ud = line_ptr(li + 1, par) + off;
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
                        if (dn_ok) d += (gc + Gd[koff(r)]) * (Ud[koff(r)] - u);
                        if (up_ok) d -= (Gu[koff(r)] + gc) * (u - Uu[koff(r)]);
                        T nm = num[r] + al * (d > T(0) ? d : T(0));
                        const T neg = al * (d < T(0) ? d : T(0));
                        T dn = (ROBUST ? den[r] : one) - neg;
                        dn = fmax(dn, gd);                 // one FMNMX (gd is not a NaN)
                        unew[j][r] = (u * nm) * frcp(dn);
                    }
                } else {
#pragma unroll
                    for (int r = 0; r < SEG; ++r) {
                        if (ROBUST) {
                            const T dn = fmax(den[r], gd);
                            unew[j][r] = (ux[r + 1] * num[r]) * frcp(dn);
                        } else {
                            unew[j][r] = ux[r + 1] * (FOLD ? num[r] * a.box_wi : num[r]);
                        }
                    }
                }
            }
            __syncwarp();
        }
        __syncthreads();
        if (last) {
            // ---- result to global, native orientation
            T *dst = a.out + frame * fsz;
#pragma unroll
            for (int j = 0; j < LPW; ++j) {
                const int li = warp + FU_WARPS * j;
                const int gl = gl0 + li;
                if (lane >= nseg) continue;
                if (!a.out_vert) {
                    T *o = dst + (int64_t)gl * n + SEG * lane;
                    if (sizeof(T) == 4) {
                        float4 *o4 = reinterpret_cast<float4 *>(o);
                        o4[0] = make_float4(unew[j][0], unew[j][1], unew[j][2], unew[j][3]);
                        o4[1] = make_float4(unew[j][4], unew[j][5], unew[j][6], unew[j][7]);
                    } else {
                        double2 *o2 = reinterpret_cast<double2 *>(o);
#pragma unroll
                        for (int i = 0; i < 4; ++i) o2[i] = make_double2(unew[j][2 * i], unew[j][2 * i + 1]);
                    }
                } else {
                    // lines are columns: stage through the (now free) own smem lines
                    T *L = own + li * ls + base0 + 9 * lane;
#pragma unroll
                    for (int r = 0; r < SEG; ++r) L[koff(r)] = unew[j][r];
                }
            }
            if (a.out_vert) {
                __syncthreads();
                // native frame [n rows][m cols]; own lines = columns gl0 .. gl0+RL-1
                for (int idx = threadIdx.x; idx < RL * n; idx += blockDim.x) {
                    const int row = idx / RL, li = idx - row * RL;
                    dst[(int64_t)row * m + gl0 + li] = own[li * ls + xaddr(HW + row)];
                }
            }
            break;
        }
        // ---- publish u': own lines + x-halos, boundary lines to the neighbours' halo[par^1]
        const int npar = par ^ 1;
#pragma unroll
        for (int j = 0; j < LPW; ++j) {
            const int li = warp + FU_WARPS * j;
            T *L = own + li * ls;
            if (lane < nseg) {
                T *P = L + base0 + 9 * lane;
#pragma unroll
                for (int r = 0; r < SEG; ++r) P[koff(r)] = unew[j][r];
            }
            __syncwarp();
            fu_fill_halo<T>(L, n, HW, a.periodic, lane);
            __syncwarp();
            if (li < 2 && nb_top)
                for (int q = lane; q < ls; q += 32) (nb_top + (RL + 4 + 2 * npar + li) * ls)[q] = L[q];
            if (li >= RL - 2 && nb_bot)
                for (int q = lane; q < ls; q += 32) (nb_bot + (RL + 2 * npar + li - RL + 2) * ls)[q] = L[q];
        }
        publish_and_g(npar);
    }
}

// launch one instantiation of k_fused_lines (cluster of a.cl CTAs per frame)
template <typename T, int R, int LPW>
cudaError_t launch_fused_t(void (*kern)(FusedKArgs<T, R>), const FusedKArgs<T, R> &a, int64_t batch,
                           cudaStream_t st, int *query_geom = nullptr) {
    constexpr int HW = HaloOf<R>::value;
    constexpr int RL = FU_WARPS * LPW;
    const size_t smem = (size_t)(2 * RL + 10 + 2 * FU_WARPS) * xline_len(a.n, HW) * sizeof(T);
    cudaError_t e = func_smem_attr((const void *)kern, smem, a.cl > 8);
    if (e != cudaSuccess) return e;
    if (a.query) {
        cudaLaunchConfig_t q = {};
        q.gridDim = dim3((unsigned)a.cl, 1, 1);
        q.blockDim = dim3(256, 1, 1);
        q.dynamicSmemBytes = smem;
        cudaLaunchAttribute qa[1];
        qa[0].id = cudaLaunchAttributeClusterDimension;
        qa[0].val.clusterDim.x = a.cl;
        qa[0].val.clusterDim.y = 1;
        qa[0].val.clusterDim.z = 1;
        q.attrs = qa;
        q.numAttrs = 1;
        e = cudaOccupancyMaxActiveClusters(a.query, kern, &q);
        if (e == cudaSuccess && query_geom) {
            query_geom[0] = a.cl;
            int per_sm = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem);
            query_geom[1] = per_sm;
        }
        return e;
    }
    const int64_t fsz = (int64_t)a.n * a.m;
    const int64_t maxf = (int64_t)(0x7fffffff / a.cl);
    for (int64_t b0 = 0; b0 < batch; b0 += maxf) {
        const int64_t nb = std::min<int64_t>(maxf, batch - b0);
        FusedKArgs<T, R> ab = a;
        ab.u0 += b0 * fsz;
        ab.fpos += b0 * fsz;
        ab.out += b0 * fsz;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(nb * a.cl), 1, 1);
        cfg.blockDim = dim3(256, 1, 1);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = a.cl;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        e = cudaLaunchKernelEx(&cfg, kern, ab);
        if (e != cudaSuccess) return e;
    }
    return cudaGetLastError();
}

// box specialisation of radius RR (md_fused_box_a.cu / md_fused_box_b.cu instantiate it)
template <typename T, int RR, int LP>
cudaError_t launch_fused_box_r(const FusedLinesArgs &d, int64_t batch, cudaStream_t st) {
    FusedKArgs<T, RR> a{};
    a.u0 = static_cast<const T *>(d.u_in);
    a.fpos = static_cast<const T *>(d.fpos);
    a.out = static_cast<T *>(d.u_out);
    a.query = d.query;
    a.n = d.n; a.m = d.m; a.iterations = d.iterations; a.out_vert = d.out_vert;
    a.periodic = d.blur.periodic;
    a.cl = d.m / (FU_WARPS * LP);
    a.alpha = T(d.alpha); a.eps_d2 = T(d.eps_d2); a.eps_r2 = T(d.eps_r2); a.has_d = d.has_d;
    a.lut = d.lut;
    a.box_wi = T(d.blur.wi);
    a.alpha_w = T(d.alpha / d.blur.wi); a.guard_w = T(kGuard / d.blur.wi); a.one_w = T(1.0 / d.blur.wi);
    if (!box_corrections<T, RR>(d.blur, d.blur.wi, a.box_cb) || !box_corrections<T, RR>(d.adj, d.blur.wi, a.box_ca))
        return cudaErrorNotSupported;
    bool corr = false;           // odd integer boxes: the plain sliding sum (no correction code)
    for (int i = 0; i < 4; ++i) corr = corr || a.box_cb[i] != T(0) || a.box_ca[i] != T(0);
    return launch_fused_t<T, RR, LP>(corr ? k_fused_lines<T, RR, LP, true, RR, true> : k_fused_lines<T, RR, LP, true, RR, false>,
                                     a, batch, st, d.query_geom);
}

// lines per warp: 4 in float (32-line CTAs, 8-CTA clusters, two CTAs per SM); for radii above 8
// the lines carry a 16-sample halo and a 32-line CTA no longer fits twice into an SM's shared
// memory (117 KB), so those run 16-line CTAs in 16-CTA clusters, again two per SM; float64: 2
template <typename T, int RR> constexpr int fused_lp() { return sizeof(T) == 8 ? 2 : (RR > 8 ? 2 : 4); }

template <typename T, int RR>
cudaError_t launch_fused_box_lpw(const FusedLinesArgs &d, int64_t batch, cudaStream_t st) {
    return launch_fused_box_r<T, RR, fused_lp<T, RR>()>(d, batch, st);
}

}  // namespace md
