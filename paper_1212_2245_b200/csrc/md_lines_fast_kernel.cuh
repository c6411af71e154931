// md_lines_fast_kernel.cuh -- the per-iteration register-window line kernel (template) and its
// launch helpers, shared by md_lines_fast.cu (dense taps) and md_lines_box_{a,b}.cu (box
// sliding sums, split over two translation units to keep compile times short).
#pragma once
#include "md_lines_fast.h"
#include "md_linefast.cuh"

namespace md {

constexpr int FTL = 8;          // lines per block
constexpr int FWARPS = 8;

__device__ __forceinline__ int wrap_or_clamp(int j, int n, int periodic) {
    // halos never exceed the extent, so one conditional wrap suffices (no integer modulo)
    if (periodic) return j < 0 ? j + n : (j >= n ? j - n : j);
    return j < 0 ? 0 : (j >= n ? n - 1 : j);
}

template <typename T>
__device__ __forceinline__ void fill_halo_line(T *line, int n, int hw, int periodic, int t, int nt) {
    for (int q = t; q < 2 * hw; q += nt) {
        const int e = q < hw ? q : n + q;                 // [0, hw) u [hw + n, n + 2hw)
        line[xaddr(e)] = line[xaddr(hw + wrap_or_clamp(e - hw, n, periodic))];
    }
}

template <typename T, int VEC> struct VecT;
template <> struct VecT<float, 4> { using type = float4; };
template <> struct VecT<double, 2> { using type = double2; };

// copy `nl` global lines (length n, contiguous) into extended smem lines
template <typename T>
__device__ __forceinline__ void load_lines(T *dst, int ls, int hw, const T *__restrict__ src, int n, int first_line,
                                           int nl, int m) {
    constexpr int V = sizeof(T) == 4 ? 4 : 2;
    using VT = typename VecT<T, V>::type;
    const int per = n / V;
    for (int idx = threadIdx.x; idx < nl * per; idx += blockDim.x) {
        const int li = idx / per, q = idx - li * per;
        const int line = first_line + li;
        if (line < 0 || line >= m) continue;
        const VT v = __ldg(reinterpret_cast<const VT *>(src + (int64_t)line * n) + q);
        T *d = dst + li * ls;
        const int e = hw + q * V;
        const T *pv = reinterpret_cast<const T *>(&v);
#pragma unroll
        for (int i = 0; i < V; ++i) d[xaddr(e + i)] = pv[i];
    }
}

template <typename T, int R, bool ROBUST, int BOXR, bool BOXC>
__global__ void __launch_bounds__(256)
k_iter_lines_fast(IterFastArgs<T, R> a) {
    constexpr int HW = HaloOf<R>::value;
    constexpr int WIN = SEG + 2 * R;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int n = a.n, m = a.m;
    const int ls = xline_len(n, HW);
    T *su = reinterpret_cast<T *>(smem_raw);       // FTL+4 lines (global l0-2 ..)
    T *sf = su + (FTL + 4) * ls;                    // FTL lines
    T *sp = sf + FTL * ls;                          // FTL lines
    T *sw = sp + FTL * ls;                          // FTL lines
    T *sg = sw + FTL * ls;                          // FTL+2 lines (global l0-1 ..)
    const int64_t fsz = (int64_t)n * m;
    const T *uin = a.u_in + blockIdx.y * fsz;
    const T *fin = a.fpos + blockIdx.y * fsz;
    T *uout = a.u_out + blockIdx.y * fsz;
    const int l0 = blockIdx.x * FTL;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nseg = n / SEG;
    const int base0 = xaddr(HW);                    // = 9*HW/8

    load_lines<T>(su, ls, HW, uin, n, l0 - 2, FTL + 4, m);
    load_lines<T>(sf, ls, HW, fin, n, l0, FTL, m);
    __syncthreads();
    for (int li = warp; li < FTL + 4; li += FWARPS) fill_halo_line<T>(su + li * ls, n, HW, a.periodic, lane, 32);
    __syncthreads();

    const T eps_r2 = a.eps_r2, eps_d2 = a.eps_d2, eps_r4 = T(4) * a.eps_r2;
    // ---- phase 1a: diffusivity g on lines l0-1 .. l0+FTL (deconv.py:191-203)
    if (a.has_d) {
        for (int gl = warp; gl < FTL + 2; gl += FWARPS) {
            const int line = l0 - 1 + gl;
            if (line < 0 || line >= m) continue;
            const bool up_ok = line > 0, dn_ok = line + 1 < m;
            for (int s = lane; s < nseg; s += 32) {
                const T *B = su + (gl + 1) * ls + base0 + 9 * s;
                T x[SEG + 2], yu[SEG], yd[SEG];
#pragma unroll
                for (int k = -1; k <= SEG; ++k) x[k + 1] = B[koff(k)];
#pragma unroll
                for (int r = 0; r < SEG; ++r) {
                    yu[r] = up_ok ? B[koff(r) - ls] : x[r + 1];
                    yd[r] = dn_ok ? B[koff(r) + ls] : x[r + 1];
                }
                T *G = sg + gl * ls + base0 + 9 * s;
#pragma unroll
                for (int r = 0; r < SEG; ++r) {
                    T dxr = x[r + 2] - x[r + 1];
                    T dxl = x[r + 1] - x[r];
                    if (r == SEG - 1 && s == nseg - 1) dxr = T(0);
                    if (r == 0 && s == 0) dxl = T(0);
                    const T dyd = yd[r] - x[r + 1], dyu = x[r + 1] - yu[r];
                    const T q = dxr * dxr + dxl * dxl + dyd * dyd + dyu * dyu;
                    // 0.5 / sqrt(q/2 + eps^2) as 1 / sqrt(2 q + 4 eps^2): bitwise the same (powers of two)
                    G[koff(r)] = frsqrt(T(2) * q + eps_r4);
                }
            }
        }
    }
    // ---- phase 1b: blur -> guard -> W, p on own lines (deconv.py:415-418, 142-162, 425-430)
    for (int li = warp; li < FTL; li += FWARPS) {
        const int line = l0 + li;
        if (line >= m) continue;
        for (int s = lane; s < nseg; s += 32) {
            const T *B = su + (li + 2) * ls + base0 + 9 * s;
            T v[WIN];
#pragma unroll
            for (int k = -R; k < SEG + R; ++k) v[k + R] = B[koff(k)];
            const T *F = sf + li * ls + base0 + 9 * s;
            T *Pp = sp + li * ls + base0 + 9 * s;
            T *Pw = sw + li * ls + base0 + 9 * s;
            T bl[SEG];
            conv_window<T, R, BOXR, BOXC>(v, a.wb, a.box_wi, a.box_cb, bl);
#pragma unroll
            for (int r = 0; r < SEG; ++r) {
                const T b = bl[r] > T(kGuard) ? bl[r] : T(kGuard);
                const T fp = F[koff(r)];
                const T rb = frcp(b);
                const T ratio = fp * rb;
                if (ROBUST) {
                    const T x = b * frcp(fp);
                    const T rr = r1_fast<T>(a.lut, x) * fp + eps_d2;
                    const T w = frsqrt(rr);       // 2 W: the 1/2 moves to alpha and the guard (phase 2)
                    Pw[koff(r)] = w;
                    Pp[koff(r)] = w * ratio;
                } else {
                    Pp[koff(r)] = ratio;
                }
            }
        }
        __syncwarp();
        fill_halo_line<T>(sp + li * ls, n, HW, a.periodic, lane, 32);
        if (ROBUST) fill_halo_line<T>(sw + li * ls, n, HW, a.periodic, lane, 32);
    }
    __syncthreads();

    // ---- phase 2: adjoint pair + TV divergence + multiplicative update (deconv.py:421-446)
    // plain integer box: adjoint window sums unscaled, 1/wi folded into alpha, the guard and
    // the unit denominator (as in k_fused_lines)
    constexpr bool FOLD = BOXR > 0 && !BOXC;
    // robust: p and W are stored as 2 W f / b and 2 W (no 1/2 multiply per pixel), so alpha and
    // the guard double -- num / den are then exactly twice the reference's (powers of two)
    constexpr int WS = ROBUST ? 2 : 1;
    const T al = (FOLD ? a.alpha_w : a.alpha) * T(WS), gd = (FOLD ? a.guard_w : T(kGuard)) * T(WS);
    const T one = FOLD ? a.one_w : T(1);
    for (int li = warp; li < FTL; li += FWARPS) {
        const int line = l0 + li;
        if (line >= m) continue;
        const bool up_ok = line > 0, dn_ok = line + 1 < m;
        for (int s = lane; s < nseg; s += 32) {
            const int off = base0 + 9 * s;
            T num[SEG], den[SEG];
            {
                const T *B = sp + li * ls + off;
                T v[WIN];
#pragma unroll
                for (int k = -R; k < SEG + R; ++k) v[k + R] = B[koff(k)];
                conv_window<T, R, BOXR, BOXC, !FOLD>(v, a.wa, a.box_wi, a.box_ca, num);
            }
            if (ROBUST) {
                const T *B = sw + li * ls + off;
                T v[WIN];
#pragma unroll
                for (int k = -R; k < SEG + R; ++k) v[k + R] = B[koff(k)];
                conv_window<T, R, BOXR, BOXC, !FOLD>(v, a.wa, a.box_wi, a.box_ca, den);
            }
            const T *U = su + (li + 2) * ls + off;
            T ux[SEG + 2];
#pragma unroll
            for (int k = -1; k <= SEG; ++k) ux[k + 1] = U[koff(k)];
            T out[SEG];
            if (a.has_d) {
                const T *G = sg + (li + 1) * ls + off;
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
                    if (dn_ok) d += (gc + G[koff(r) + ls]) * (U[koff(r) + ls] - u);
                    if (up_ok) d -= (G[koff(r) - ls] + gc) * (u - U[koff(r) - ls]);
                    const T nm = num[r] + al * (d > T(0) ? d : T(0));
                    const T neg = al * (d < T(0) ? d : T(0));
                    T dn = (ROBUST ? den[r] : one) - neg;
                    dn = fmax(dn, gd);
                    out[r] = (u * nm) * frcp(dn);
                }
            } else {
#pragma unroll
                for (int r = 0; r < SEG; ++r) {
                    const T u = ux[r + 1];
                    if (ROBUST) {
                        const T dn = fmax(den[r], gd);
                        out[r] = (u * num[r]) * frcp(dn);
                    } else {
                        out[r] = u * (FOLD ? num[r] * a.box_wi : num[r]);
                    }
                }
            }
            T *dst = uout + (int64_t)line * n + SEG * s;
            if (sizeof(T) == 4) {
                float4 *d4 = reinterpret_cast<float4 *>(dst);
                d4[0] = make_float4(out[0], out[1], out[2], out[3]);
                d4[1] = make_float4(out[4], out[5], out[6], out[7]);
            } else {
                double2 *d2 = reinterpret_cast<double2 *>(dst);
#pragma unroll
                for (int i = 0; i < 4; ++i) d2[i] = make_double2(out[2 * i], out[2 * i + 1]);
            }
        }
    }
}

template <typename T, int R>
size_t iter_fast_smem(int n) {
    constexpr int HW = HaloOf<R>::value;
    return (size_t)(5 * FTL + 6) * xline_len(n, HW) * sizeof(T);
}

template <typename T, int R>
cudaError_t launch_iter_fast_k(void (*kern)(IterFastArgs<T, R>), const IterFastArgs<T, R> &a, int64_t batch,
                               cudaStream_t st) {
    const size_t smem = iter_fast_smem<T, R>(a.n);
    cudaError_t e = func_smem_attr((const void *)kern, smem);
    if (e != cudaSuccess) return e;
    const int tiles = (a.m + FTL - 1) / FTL;
    const int64_t fsz = (int64_t)a.n * a.m;
    for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
        const int nb = (int)((batch - b0) < 65535 ? (batch - b0) : 65535);
        IterFastArgs<T, R> ab = a;
        ab.u_in += b0 * fsz;
        ab.fpos += b0 * fsz;
        ab.u_out += b0 * fsz;
        kern<<<dim3(tiles, nb), 256, smem, st>>>(ab);
    }
    return cudaGetLastError();
}

// box specialisation of radius RR (md_lines_box_a.cu / md_lines_box_b.cu instantiate it)
template <typename T, int RR>
cudaError_t launch_iter_fast_box_r(const IterFastDesc &d, int64_t batch, cudaStream_t st) {
    IterFastArgs<T, RR> a{};
    a.u_in = static_cast<const T *>(d.u_in);
    a.fpos = static_cast<const T *>(d.fpos);
    a.u_out = static_cast<T *>(d.u_out);
    a.n = d.n; a.m = d.m; a.periodic = d.blur.periodic;
    a.alpha = T(d.alpha); a.eps_d2 = T(d.eps_d2); a.eps_r2 = T(d.eps_r2); a.has_d = d.has_d;
    a.lut = d.lut;
    a.box_wi = T(d.blur.wi);
    a.alpha_w = T(d.alpha / d.blur.wi); a.guard_w = T(kGuard / d.blur.wi); a.one_w = T(1.0 / d.blur.wi);
    if (!box_corrections<T, RR>(d.blur, d.blur.wi, a.box_cb) || !box_corrections<T, RR>(d.adj, d.blur.wi, a.box_ca))
        return cudaErrorNotSupported;
    bool corr = false;           // odd integer boxes: the plain sliding sum
    for (int i = 0; i < 4; ++i) corr = corr || a.box_cb[i] != T(0) || a.box_ca[i] != T(0);
    return launch_iter_fast_k<T, RR>(corr ? k_iter_lines_fast<T, RR, true, RR, true> : k_iter_lines_fast<T, RR, true, RR, false>,
                                     a, batch, st);
}

}  // namespace md
