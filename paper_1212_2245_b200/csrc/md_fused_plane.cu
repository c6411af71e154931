// md_fused_plane.cu -- the whole RRRL iteration loop for small frames blurred by a 2D PSF
// (FOURIER_2D with direct periodic taps, or the clamped spatial convolver), resident in the
// distributed shared memory of one thread-block cluster per frame.
//
// Replaces the per-iteration k_plane_a_fast / k_plane_b_fast pair (md_plane_fast.cu) -- i.e.
// _iterate_rrrl (deconv.py:512-521) with _FourierConvolver2D / _SpatialConvolver, the weight
// arrays (142-162), the diffusion term (187-213) and _combine (421-446) -- when a frame fits
// on the cluster: no iterate, p or W ever leaves the chip between the Wiener init and the
// final store.
//
// Geometry: CTA `rank` of a CL-CTA cluster owns RL = H / CL consecutive rows (RL <= 32) of
// width W = 32 J; warp w owns the row pair (2w, 2w + 1), lane l the J columns x = l + 32 j of
// both rows, so consecutive lanes hit consecutive banks. Rows carry an x-halo of HX columns
// (wrapped or edge-replicated). Taps are regrouped on the host into COLUMNS (fixed dx, a run
// of consecutive dy): walking a column downwards, every loaded value feeds the upper row with
// tap i and the lower row with tap i - 1, so a row pair costs len + 1 shared loads per column
// instead of 2 len -- the direct convolution is bound by the shared-memory pipe, not the FMAs.
// p and W are stored interleaved (one 8-byte load feeds both halves of the adjoint pair).
//
// Per iteration (U: iterate rows with halos; PW: (p, W) rows with halos; G: diffusivity):
//   A: own rows: b = taps(U) -> (p, W) (+ x-halo) || G rows -1..RL, stash U rows -1, RL
//      push own boundary PW rows into the neighbours' PW halos       | cluster barrier 1
//   B: own rows: (num, den) = taps(PW); D from G + U (+ stash) -> u' (registers)
//      u' -> own U rows; push boundary rows into the neighbours' U halos | cluster barrier 2
// The stash lets a neighbour overwrite this CTA's U halo while it is still in stage B, so two
// cluster barriers per iteration suffice. Without a y-period the image-edge halos are
// replicated locally (clamped convolver), matching pf_resolve in md_plane_fast.cu.
#include <cooperative_groups.h>

#include <algorithm>

#include "md_coltaps.cuh"
#include "md_fused_plane.h"
#include "md_linefast.cuh"

namespace cg = cooperative_groups;

namespace md {

// warps per row pair: 2 (column halves, 1024 threads at 64 registers) hides more latency but
// halves the columns that amortise each tap's loop overhead -- measured slower than 1
constexpr int FP_SPLIT = 1;
constexpr int FP_WARPS = 16 * FP_SPLIT;
constexpr int FP_THREADS = FP_WARPS * 32;
constexpr int FP_MAXRL = 2 * FP_WARPS / FP_SPLIT;   // one row pair per FP_SPLIT warps
constexpr int FP_MAXHX = 32;                    // x-halo sources lie in the first / last 32 columns
template <typename T> struct FusedPlaneKArgs {
    const T *u0, *fpos;
    T *out;
    int H, W, rl, cl, periodic, iterations;
    int hx, rs;          // x-halo columns, row stride (elements of the row's field)
    int ut, ub;          // U halo rows above / below
    int pt, pb;          // PW halo rows above / below
    ColTaps<T> tb, ta;   // blur taps over U, adjoint taps over PW
    T alpha, eps_d2, eps_r2;
    int has_d;
    LutView lut;
};

// shared-memory layout (offsets in elements of T), identical in every CTA of the cluster
struct FpLayout {
    int u, pw, g, stash, total;
};

__host__ __device__ inline FpLayout fp_layout(int rl, int rs, int W, int ut, int ub, int pt, int pb) {
    FpLayout L;
    L.u = 0;
    L.pw = L.u + (rl + ut + ub) * rs;
    L.g = L.pw + 2 * (rl + pt + pb) * rs;
    L.stash = L.g + (rl + 2) * rs;
    L.total = L.stash + 2 * W;
    return L;
}

__device__ __forceinline__ int fp_wrap(int c, int n, int periodic) {
    if (periodic) return c < 0 ? c + n : (c >= n ? c - n : c);
    return c < 0 ? 0 : (c >= n ? n - 1 : c);
}

// store a warp's JW values of one row (row points at column -hx; this warp holds the columns
// x = lane + 32 (jj0 + j)) together with the x-halo copies they source: with a period the left
// halo mirrors the last hx columns and the right halo the first hx, without one the halos
// replicate the edge columns (hx <= 32, so only the first / last column block feeds a halo)
template <typename E, int JW>
__device__ __forceinline__ void fp_store_row(E *row, const E (&v)[JW], int lane, int jj0, int W, int hx,
                                             int periodic) {
#pragma unroll
    for (int j = 0; j < JW; ++j) row[hx + lane + 32 * (jj0 + j)] = v[j];
    const int nb = W >> 5;
    if (jj0 == 0) {                                    // first block: x = lane
        if (periodic) {
            if (lane < hx) row[hx + W + lane] = v[0];
        } else if (lane == 0) {
            for (int q = 0; q < hx; ++q) row[q] = v[0];
        }
    }
    if (jj0 + JW == nb) {                              // last block: x = W - 32 + lane
        const int x = W - 32 + lane;
        if (periodic) {
            if (x >= W - hx) row[hx + x - W] = v[JW - 1];
        } else if (lane == 31) {
            for (int q = 0; q < hx; ++q) row[hx + W + q] = v[JW - 1];
        }
    }
}

// 16-byte block copy (rows are 16-byte aligned), block-collective
__device__ __forceinline__ void fp_copy(void *dst, const void *src, int bytes) {
    int4 *d = static_cast<int4 *>(dst);
    const int4 *s = static_cast<const int4 *>(src);
    for (int i = threadIdx.x; i < bytes / 16; i += blockDim.x) d[i] = s[i];
}

__device__ __forceinline__ void fp_cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

template <typename T, int J, bool ROBUST>
__global__ void __launch_bounds__(FP_THREADS, 1)
k_fused_plane(FusedPlaneKArgs<T> a) {
    using T2 = typename Vec2<T>::type;
    constexpr int JW = J / FP_SPLIT;         // column blocks per warp
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T *sm = reinterpret_cast<T *>(smem_raw);
    const int H = a.H, W = a.W, RL = a.rl, rs = a.rs, hx = a.hx;
    const int CL = a.cl;
    const int rank = (int)cluster.block_rank();
    const int64_t frame = blockIdx.x / CL;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int jj0 = (warp % FP_SPLIT) * JW;  // this warp's column blocks
    const int xl = lane + 32 * jj0;          // its first column
    const int gy0 = rank * RL;
    const int64_t fsz = (int64_t)H * W;
    const T *fpos = a.fpos + frame * fsz;
    const FpLayout L = fp_layout(RL, rs, W, a.ut, a.ub, a.pt, a.pb);
    const int ut = a.ut, ub = a.ub, pt = a.pt, pb = a.pb;
    poison_smem(smem_raw);
    MD_CHECK((size_t)L.total * sizeof(T) <= dyn_smem_bytes() && RL * CL == H && (RL & 1) == 0);
    auto urow = [&](T *base, int r) {
        MD_CHECK(r >= -ut && r < RL + ub);
        return base + L.u + (r + ut) * rs;
    };
    auto pwrow = [&](T *base, int r) {
        MD_CHECK(r >= -pt && r < RL + pb);
        return reinterpret_cast<T2 *>(base + L.pw) + (r + pt) * rs;
    };
    T *G = sm + L.g + rs;                    // row r at G + r * rs, r in [-1, RL]
    T *stash = sm + L.stash;                 // U rows -1 and RL, columns 0..W-1

    // neighbours in the row ring; without a y-period the image edges have none
    const bool has_up = a.periodic || rank > 0, has_dn = a.periodic || rank < CL - 1;
    cluster.sync();                          // all CTAs resident before DSMEM traffic
    T *nb_up = has_up ? cluster.map_shared_rank(sm, (rank + CL - 1) % CL) : nullptr;
    T *nb_dn = has_dn ? cluster.map_shared_rank(sm, (rank + 1) % CL) : nullptr;

    // boundary rows of a field (rows [-top, RL + bot) around own rows) to the neighbours, or
    // edge replication at an image edge without a y-period
    auto push_rows = [&](auto rowf, int top, int bot, int rbytes) {
        if (nb_up) fp_copy(rowf(nb_up, RL), rowf(sm, 0), bot * rbytes);          // its bottom halo
        else for (int r = 1; r <= top; ++r) fp_copy(rowf(sm, -r), rowf(sm, 0), rbytes);
        if (nb_dn) fp_copy(rowf(nb_dn, -top), rowf(sm, RL - top), top * rbytes);  // its top halo
        else for (int r = 0; r < bot; ++r) fp_copy(rowf(sm, RL + r), rowf(sm, RL - 1), rbytes);
    };
    const int ubytes = rs * (int)sizeof(T), pwbytes = rs * (int)sizeof(T2);

    const int r0 = 2 * (warp / FP_SPLIT);    // this warp's row pair
    const bool pair = r0 < RL;
    // ---- u0: own rows + x-halos, then the halos of the neighbours
    if (pair) {
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const T *src = a.u0 + frame * fsz + (int64_t)(gy0 + r0 + k) * W + xl;
            T v[JW];
#pragma unroll
            for (int j = 0; j < JW; ++j) v[j] = src[32 * j];
            fp_store_row<T, JW>(urow(sm, r0 + k), v, lane, jj0, W, hx, a.periodic);
        }
    }
    __syncthreads();
    push_rows(urow, ut, ub, ubytes);
    fp_cluster_sync();

    const T eps_d2 = a.eps_d2, eps_r2 = a.eps_r2, alpha = a.alpha;
    for (int it = 0; it < a.iterations; ++it) {
        const bool last = it == a.iterations - 1;
        // ---- stage A: blur -> (p, W) on own rows
        if (pair) {
            T b[2][JW];
            col_taps_pair<T, JW, 32>(urow(sm, r0) + hx + xl, rs, a.tb, b[0], b[1]);
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const T *F = fpos + (int64_t)(gy0 + r0 + k) * W + xl;
                T2 v[JW];
#pragma unroll
                for (int j = 0; j < JW; ++j) {
                    const T bb = b[k][j] > T(kGuard) ? b[k][j] : T(kGuard);
                    const T fv = __ldg(F + 32 * j);
                    const T ratio = fv * frcp(bb);
                    if (ROBUST) {
                        const T wv = T(0.5) * frsqrt(r1_fast<T>(a.lut, bb * frcp(fv)) * fv + eps_d2);
                        v[j].x = wv * ratio;
                        v[j].y = wv;
                    } else {
                        v[j].x = ratio;
                        v[j].y = T(0);
                    }
                }
                fp_store_row<T2, JW>(pwrow(sm, r0 + k), v, lane, jj0, W, hx, a.periodic);
            }
        }
        // ---- diffusivity on rows -1..RL (deconv.py:191-203); Neumann at the image border
        if (a.has_d) {
            for (int u = warp; u < FP_SPLIT * (RL + 2); u += FP_WARPS) {
                const int r = u / FP_SPLIT - 1;
                const int gy = gy0 + r;
                if (gy < 0 || gy >= H) continue;
                const T *c = urow(sm, r) + hx;
                const bool up_ok = gy > 0, dn_ok = gy + 1 < H;
                const int x0 = lane + 32 * ((u % FP_SPLIT) * JW);
#pragma unroll
                for (int j = 0; j < JW; ++j) {
                    const int x = x0 + 32 * j;
                    const T c0 = c[x];
                    T dr = c[x + 1] - c0, dl = c0 - c[x - 1];
                    if (x + 1 >= W) dr = T(0);
                    if (x == 0) dl = T(0);
                    const T dd = dn_ok ? c[x + rs] - c0 : T(0);
                    const T du = up_ok ? c0 - c[x - rs] : T(0);
                    const T q = dr * dr + dl * dl + dd * dd + du * du;
                    G[r * rs + hx + x] = T(0.5) * frsqrt(T(0.5) * q + eps_r2);
                }
            }
            // rows -1 and RL of U: stage B reads them after the neighbours may have moved on
            for (int i = threadIdx.x; i < 2 * W; i += blockDim.x) {
                const int k = i >= W, x = i - k * W;
                stash[i] = urow(sm, k ? RL : -1)[hx + x];
            }
        }
        __syncthreads();
        push_rows(pwrow, pt, pb, pwbytes);
        fp_cluster_sync();

        // ---- stage B: adjoint pair + TV + multiplicative update (registers)
        T unew[2][JW];
        if (pair) {
            T num[2][JW], den[2][JW];
            col_taps_pair2<T, JW, 32>(pwrow(sm, r0) + hx + xl, rs, a.ta, num[0], num[1], den[0], den[1]);
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int r = r0 + k;
                const int gy = gy0 + r;
                const T *U = urow(sm, r) + hx;
                const T *Uu = r > 0 ? U - rs : stash;
                const T *Ud = r < RL - 1 ? U + rs : stash + W;
                const T *Gr = G + r * rs + hx;
                const bool up_ok = gy > 0, dn_ok = gy + 1 < H;
#pragma unroll
                for (int j = 0; j < JW; ++j) {
                    const int x = xl + 32 * j;
                    const T uv = U[x];
                    T nm = num[k][j];
                    T dn = ROBUST ? den[k][j] : T(1);
                    if (a.has_d) {
                        const T gc = Gr[x];
                        T d = T(0);
                        if (x + 1 < W) d += (gc + Gr[x + 1]) * (U[x + 1] - uv);
                        if (x > 0) d -= (Gr[x - 1] + gc) * (uv - U[x - 1]);
                        if (dn_ok) d += (gc + Gr[x + rs]) * (Ud[x] - uv);
                        if (up_ok) d -= (Gr[x - rs] + gc) * (uv - Uu[x]);
                        nm += alpha * (d > T(0) ? d : T(0));
                        dn -= alpha * (d < T(0) ? d : T(0));
                    }
                    if (ROBUST || a.has_d) {
                        dn = dn > T(kGuard) ? dn : T(kGuard);
                        unew[k][j] = (uv * nm) * frcp(dn);
                    } else {
                        unew[k][j] = uv * nm;
                    }
                }
            }
        }
        __syncthreads();
        if (last) {
            if (pair) {
                T *dst = a.out + frame * fsz + (int64_t)(gy0 + r0) * W + xl;
#pragma unroll
                for (int k = 0; k < 2; ++k)
#pragma unroll
                    for (int j = 0; j < JW; ++j) dst[(int64_t)k * W + 32 * j] = unew[k][j];
            }
            break;
        }
        if (pair) {
#pragma unroll
            for (int k = 0; k < 2; ++k) fp_store_row<T, JW>(urow(sm, r0 + k), unew[k], lane, jj0, W, hx, a.periodic);
        }
        __syncthreads();
        push_rows(urow, ut, ub, ubytes);
        fp_cluster_sync();
    }
}

// ---------------------------------------------------------------------------------- host

namespace {

struct FpGeom {
    int cl, rl, hx, rs, ut, ub, pt, pb;
    size_t smem;
};

#ifndef MD_FP_MINCL
#define MD_FP_MINCL 2
#endif

bool fp_geometry(int H, int W, const PlaneHalo &hb, const PlaneHalo &ha, int dtype, FpGeom *g) {
    if (W != 64 && W != 128 && W != 256) return false;
    const int es = dtype == 0 ? 8 : 4;
    const int hxn = std::max(std::max(hb.hl, hb.hr), std::max(ha.hl, ha.hr));
    const int hx = (hxn + 3) & ~3;                      // rows stay 16-byte aligned
    if (hx > FP_MAXHX || hx > W / 2) return false;
    const int rs = W + 2 * hx;
    const int ut = std::max(hb.ht, 2), ub = std::max(hb.hb, 2);
    for (int cl = MD_FP_MINCL; cl <= 16; cl *= 2) {
        if (H % cl) continue;
        const int rl = H / cl;
        if (rl > FP_MAXRL || (rl & 1)) continue;
        if (std::max(ut, ub) > rl || std::max(ha.ht, ha.hb) > rl) continue;
        const FpLayout L = fp_layout(rl, rs, W, ut, ub, ha.ht, ha.hb);
        const size_t smem = (size_t)L.total * es;
        if (smem > 227 * 1024) continue;
        *g = FpGeom{cl, rl, hx, rs, ut, ub, ha.ht, ha.hb, smem};
        return true;
    }
    return false;
}

template <typename T, int J>
cudaError_t launch_j(const FusedPlaneDesc &d, const FpGeom &g, int64_t batch, cudaStream_t st) {
    FusedPlaneKArgs<T> a{};
    a.u0 = static_cast<const T *>(d.u0);
    a.fpos = static_cast<const T *>(d.fpos);
    a.out = static_cast<T *>(d.u_out);
    a.H = d.H; a.W = d.W; a.rl = g.rl; a.cl = g.cl; a.periodic = d.periodic; a.iterations = d.iterations;
    a.hx = g.hx; a.rs = g.rs; a.ut = g.ut; a.ub = g.ub; a.pt = g.pt; a.pb = g.pb;
    if (!build_col_taps<T>(*d.taps_blur, g.rs, &a.tb) || !build_col_taps<T>(*d.taps_adj, g.rs, &a.ta))
        return cudaErrorNotSupported;
    a.alpha = T(d.alpha); a.eps_d2 = T(d.eps_d2); a.eps_r2 = T(d.eps_r2); a.has_d = d.has_d;
    a.lut = d.lut;
    auto kern = d.robust ? k_fused_plane<T, J, true> : k_fused_plane<T, J, false>;
    cudaError_t e = func_smem_attr((const void *)kern, g.smem, g.cl > 8);
    if (e != cudaSuccess) return e;
    const int64_t fsz = (int64_t)d.H * d.W;
    const int64_t maxf = (int64_t)(0x7fffffff / g.cl);
    for (int64_t b0 = 0; b0 < batch; b0 += maxf) {
        const int64_t nb = std::min<int64_t>(maxf, batch - b0);
        FusedPlaneKArgs<T> ab = a;
        ab.u0 += b0 * fsz;
        ab.fpos += b0 * fsz;
        ab.out += b0 * fsz;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(nb * g.cl), 1, 1);
        cfg.blockDim = dim3(FP_THREADS, 1, 1);
        cfg.dynamicSmemBytes = g.smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = g.cl;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        e = cudaLaunchKernelEx(&cfg, kern, ab);
        if (e != cudaSuccess) return e;
    }
    return cudaGetLastError();
}

}  // namespace

bool fused_plane_supported(int H, int W, const PlaneHalo &hb, const PlaneHalo &ha,
                           const std::vector<PlaneTap> &taps_blur, const std::vector<PlaneTap> &taps_adj, int dtype) {
    FpGeom g;
    if (!fp_geometry(H, W, hb, ha, dtype, &g)) return false;
    return dtype == 0 ? build_col_taps<double>(taps_blur, g.rs, nullptr) && build_col_taps<double>(taps_adj, g.rs, nullptr)
                      : build_col_taps<float>(taps_blur, g.rs, nullptr) && build_col_taps<float>(taps_adj, g.rs, nullptr);
}

template <typename T>
cudaError_t launch_fused_plane(const FusedPlaneDesc &d, int64_t batch, cudaStream_t st) {
    FpGeom g;
    if (!fp_geometry(d.H, d.W, d.hb, d.ha, sizeof(T) == 8 ? 0 : 1, &g)) return cudaErrorNotSupported;
    if (d.W == 64) return launch_j<T, 2>(d, g, batch, st);
    if (d.W == 128) return launch_j<T, 4>(d, g, batch, st);
    return launch_j<T, 8>(d, g, batch, st);
}

template cudaError_t launch_fused_plane<double>(const FusedPlaneDesc &, int64_t, cudaStream_t);
template cudaError_t launch_fused_plane<float>(const FusedPlaneDesc &, int64_t, cudaStream_t);

}  // namespace md
