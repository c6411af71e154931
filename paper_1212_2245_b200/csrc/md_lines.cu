// md_lines.cu -- kernels for 1D blur (Scenario.BOX_1D / FOURIER_1D and 1D PSFs under the
// spatial / fourier convolver modes).
//
// Internal layout: "line-major" -- every line along the blur axis is contiguous,
// [batch][m lines][n samples]. Horizontal blur is the native layout; vertical blur is
// transposed by the first kernel (k_wiener_lines / k_init_lines) and back by the last one,
// mirroring the reference's canonical vertical orientation (deconv.py:624-628, 657, 683).
//
//   k_wiener_lines  per line pair: FFT (DIF) -> x Wiener multiplier -> IFFT (DIT) -> clamp.
//                   Replaces FourierPlan._run / apply_column_filter / _wiener_multiplier
//                   (fft.py:87-107, 236-258; deconv.py:253-254, 666-672).
//   k_iter_lines    ONE launch per RRRL iteration over a tile of TL full lines:
//                   blur (sliding-window box or register-blocked taps, clamped or periodic)
//                   -> robust weight W -> p = W f/b -> adjoint pair -> TV divergence D
//                   (2-line halo) -> multiplicative update. Replaces _iterate_rrrl and its
//                   callees (deconv.py:142-213, 415-446, 512-521; conv.py:141-173).
#include "md_fft.cuh"
#include "md_internal.h"

namespace md {

// padded shared-memory index: one spare element every 32 words so that the run-per-thread
// access pattern (8 consecutive samples per thread) is bank-conflict free
template <typename T> __device__ __forceinline__ int pidx(int j) {
    return sizeof(T) == 8 ? j + (j >> 4) : j + (j >> 5);
}
template <typename T> __host__ __device__ inline int padded_len(int n) {
    return sizeof(T) == 8 ? n + (n >> 4) + 2 : n + (n >> 5) + 2;
}

__device__ __forceinline__ int resolve(int k, int n, int periodic) {
    if (periodic) {
        k %= n;
        return k < 0 ? k + n : k;
    }
    return k < 0 ? 0 : (k >= n ? n - 1 : k);
}

// --------------------------------------------------------------------------------------
// Wiener per line pair (1D)

template <typename T>
__global__ void __launch_bounds__(256)
k_wiener_lines(WienerLinesArgs a) {
    using C = cx_t<T>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int n = a.n, m = a.m, LP = a.lp;
    const int cs = fline_stride<sizeof(C)>(n);                         // complex line stride (md_fft.cuh padding)
    C *s = reinterpret_cast<C *>(smem_raw);
    T *sfr = reinterpret_cast<T *>(s + LP * cs);             // raw f (only when in_vert)
    const int P = padded_len<T>(n);
    const int64_t fr = blockIdx.y;
    const T *in = static_cast<const T *>(a.in) + fr * (int64_t)n * m;
    T *out = static_cast<T *>(a.out) + fr * (int64_t)n * m;
    T *fpos = a.fpos ? static_cast<T *>(a.fpos) + fr * (int64_t)n * m : nullptr;
    const int L0 = 2 * LP * blockIdx.x;
    const int NL = 2 * LP;
    const T floor = T(a.floor);

    for (int idx = threadIdx.x; idx < NL * n; idx += blockDim.x) {
        int li, j;
        if (a.in_vert) { j = idx / NL; li = idx - j * NL; }
        else { li = idx / n; j = idx - li * n; }
        const int line = L0 + li;
        T v = T(0);
        if (line < m) {
            v = a.in_vert ? in[(int64_t)j * m + line] : in[(int64_t)line * n + j];
            if (fpos) {
                if (a.in_vert) sfr[li * P + pidx<T>(j)] = v;
                else fpos[(int64_t)line * n + j] = v > floor ? v : floor;
            }
        }
        C *c = s + (li >> 1) * cs + fpad<sizeof(C)>(j);
        if (li & 1) c->y = v; else c->x = v;
    }
    __syncthreads();
    if (a.log2n > 0) fft_dif_lines(s, a.log2n, LP, cs, static_cast<const C *>(a.tw));
    const C *mult = static_cast<const C *>(a.mult);
    for (int idx = threadIdx.x; idx < LP * n; idx += blockDim.x) {
        const int l = idx / n, p = idx - l * n;
        s[l * cs + fpad<sizeof(C)>(p)] = cmul(s[l * cs + fpad<sizeof(C)>(p)], __ldg(mult + p));
    }
    __syncthreads();
    if (a.log2n > 0) fft_dit_inv_lines(s, a.log2n, LP, cs, static_cast<const C *>(a.tw));
    const T inv_n = T(1) / T(n);
    for (int idx = threadIdx.x; idx < NL * n; idx += blockDim.x) {
        int li, j;
        if (a.out_vert) { j = idx / NL; li = idx - j * NL; }
        else { li = idx / n; j = idx - li * n; }
        const int line = L0 + li;
        if (line >= m) continue;
        const C c = s[(li >> 1) * cs + fpad<sizeof(C)>(j)];
        T v = ((li & 1) ? c.y : c.x) * inv_n;
        if (a.clamp) v = v > floor ? v : floor;
        if (a.out_vert) out[(int64_t)j * m + line] = v;
        else out[(int64_t)line * n + j] = v;
    }
    if (fpos && a.in_vert) {
        for (int idx = threadIdx.x; idx < NL * n; idx += blockDim.x) {
            const int li = idx / n, j = idx - li * n;
            const int line = L0 + li;
            if (line >= m) continue;
            const T v = sfr[li * P + pidx<T>(j)];
            fpos[(int64_t)line * n + j] = v > floor ? v : floor;
        }
    }
}

// --------------------------------------------------------------------------------------
// line convolution on a shared-memory line: RUN consecutive outputs per thread

constexpr int RUN = 8;

// a * b + c as the reference's NumPy rounds it (two roundings) when EXACT, else contracted
template <bool EXACT>
__device__ __forceinline__ double madd(double a, double b, double c) {
    return EXACT ? __dadd_rn(__dmul_rn(a, b), c) : a * b + c;
}
template <bool EXACT>
__device__ __forceinline__ float madd(float a, float b, float c) { return a * b + c; }

// EXACT: the public convolve path (synth_blur / convolve_array, conv.py:85-116), which must
// reproduce the reference's rounding so quantised synthetic inputs match bit for bit
template <typename T, bool EXACT = false>
__device__ __forceinline__ void conv_run(const T *line, int n, int j0, const LineConv &c,
                                         const T *taps, T out[RUN]) {
    const int per = c.periodic;
    if (c.kind == LINE_BOX) {
        const T wi = T(c.wi), we = T(c.we);
        T s = T(0);
        for (int k = c.lo; k <= c.hi; ++k) s += line[pidx<T>(resolve(j0 + k, n, per))];
#pragma unroll
        for (int r = 0; r < RUN; ++r) {
            if (r > 0) s += line[pidx<T>(resolve(j0 + r + c.hi, n, per))] -
                            line[pidx<T>(resolve(j0 + r - 1 + c.lo, n, per))];
            T v = s * wi;
            if (c.ends) {
                v += we * line[pidx<T>(resolve(j0 + r + c.elo, n, per))];
                v += we * line[pidx<T>(resolve(j0 + r + c.ehi, n, per))];
            }
            out[r] = v;
        }
    } else {
        // out[j] = sum_t w[t] * a[j + c - t], taps accumulated in index order (conv.py:108-116)
#pragma unroll
        for (int r = 0; r < RUN; ++r) out[r] = T(0);
        for (int t = 0; t < c.ntaps; ++t) {
            const T w = taps[t];
            if (w == T(0)) continue;
            const int base = j0 + c.center - t;
#pragma unroll
            for (int r = 0; r < RUN; ++r) out[r] = madd<EXACT>(w, line[pidx<T>(resolve(base + r, n, per))], out[r]);
        }
    }
}

// --------------------------------------------------------------------------------------
// one fused RRRL iteration over TL full lines (+2-line halo for the TV stencil)

template <typename T, bool ROBUST>
__global__ void __launch_bounds__(256)
k_iter_lines(IterLinesArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int n = a.n, m = a.m, TL = a.tl;
    const int P = padded_len<T>(n);
    T *su = reinterpret_cast<T *>(smem_raw);          // (TL+4) lines: l0-2 .. l0+TL+1
    T *sf = su + (TL + 4) * P;                         // TL lines, floored observation
    T *sp = sf + TL * P;                               // W f / b   (or f / b for RL)
    T *sw = sp + TL * P;                               // W
    T *sg = sw + TL * P;                               // (TL+2) lines: diffusivity g
    T *stap = sg + (TL + 2) * P;                       // blur taps, then adjoint taps
    const int64_t fr = blockIdx.y;
    const int64_t fsz = (int64_t)n * m;
    const T *uin = static_cast<const T *>(a.u_in) + fr * fsz;
    const T *fin = static_cast<const T *>(a.fpos) + fr * fsz;
    T *uout = static_cast<T *>(a.u_out) + fr * fsz;
    const int l0 = blockIdx.x * TL;
    const bool has_d = a.has_d;

    for (int t = threadIdx.x; t < a.blur.ntaps; t += blockDim.x) stap[t] = T(a.taps_blur[t]);
    for (int t = threadIdx.x; t < a.adj.ntaps; t += blockDim.x) stap[a.blur.ntaps + t] = T(a.taps_adj[t]);
    const int ulines = has_d ? TL + 4 : TL;
    const int uoff = has_d ? 0 : 2;
    for (int idx = threadIdx.x; idx < ulines * n; idx += blockDim.x) {
        const int li = idx / n, j = idx - li * n;
        const int line = l0 - 2 + uoff + li;
        if (line >= 0 && line < m) su[(li + uoff) * P + pidx<T>(j)] = uin[(int64_t)line * n + j];
    }
    for (int idx = threadIdx.x; idx < TL * n; idx += blockDim.x) {
        const int li = idx / n, j = idx - li * n;
        const int line = l0 + li;
        if (line < m) sf[li * P + pidx<T>(j)] = fin[(int64_t)line * n + j];
    }
    __syncthreads();

    const int runs = (n + RUN - 1) / RUN;
    const T eps_d2 = T(a.eps_d2), eps_r2 = T(a.eps_r2);
    // phase 1: diffusivity on lines l0-1 .. l0+TL and blur -> W, p on own lines
    if (has_d) {
        for (int q = threadIdx.x; q < (TL + 2) * runs; q += blockDim.x) {
            const int gl = q / runs, j0 = (q - gl * runs) * RUN;
            const int line = l0 - 1 + gl;
            if (line < 0 || line >= m) continue;
            const T *row = su + (gl + 1) * P;
            const T *up = su + gl * P;         // line - 1
            const T *dn = su + (gl + 2) * P;   // line + 1
            for (int r = 0; r < RUN; ++r) {
                const int j = j0 + r;
                if (j >= n) break;
                const T c = row[pidx<T>(j)];
                T q2 = T(0);
                if (j + 1 < n) { const T d = row[pidx<T>(j + 1)] - c; q2 += d * d; }
                if (j > 0) { const T d = c - row[pidx<T>(j - 1)]; q2 += d * d; }
                if (line + 1 < m) { const T d = dn[pidx<T>(j)] - c; q2 += d * d; }
                if (line > 0) { const T d = c - up[pidx<T>(j)]; q2 += d * d; }
                sg[gl * P + pidx<T>(j)] = T(0.5) / sqrt(T(0.5) * q2 + eps_r2);
            }
        }
    }
    for (int q = threadIdx.x; q < TL * runs; q += blockDim.x) {
        const int li = q / runs, j0 = (q - li * runs) * RUN;
        if (l0 + li >= m) continue;
        T b[RUN];
        conv_run<T>(su + (li + 2) * P, n, j0, a.blur, stap, b);
#pragma unroll
        for (int r = 0; r < RUN; ++r) {
            const int j = j0 + r;
            if (j < n) {
                const T bb = b[r] > T(kGuard) ? b[r] : T(kGuard);
                const T fp = sf[li * P + pidx<T>(j)];
                const T ratio = fp / bb;
                if (ROBUST) {
                    const T w = robust_weight_floored<T>(a.lut, fp, bb, eps_d2);
                    sw[li * P + pidx<T>(j)] = w;
                    sp[li * P + pidx<T>(j)] = w * ratio;
                } else {
                    sp[li * P + pidx<T>(j)] = ratio;
                }
            }
        }
    }
    __syncthreads();

    // phase 2: adjoint pair, TV divergence, multiplicative update
    const T alpha = T(a.alpha);
    const T *tap_adj = stap + a.blur.ntaps;
    for (int q = threadIdx.x; q < TL * runs; q += blockDim.x) {
        const int li = q / runs, j0 = (q - li * runs) * RUN;
        const int line = l0 + li;
        if (line >= m) continue;
        T num[RUN], den[RUN];
        conv_run<T>(sp + li * P, n, j0, a.adj, tap_adj, num);
        if (ROBUST) conv_run<T>(sw + li * P, n, j0, a.adj, tap_adj, den);
        const T *row = su + (li + 2) * P;
        const T *up = su + (li + 1) * P;
        const T *dn = su + (li + 3) * P;
        const T *g = sg + (li + 1) * P;
        const T *gu = sg + li * P;
        const T *gd = sg + (li + 2) * P;
#pragma unroll
        for (int r = 0; r < RUN; ++r) {
            const int j = j0 + r;
            if (j >= n) break;
            const T u = row[pidx<T>(j)];
            T d = T(0);
            if (has_d) {
                const T gc = g[pidx<T>(j)];
                if (j + 1 < n) d += (gc + g[pidx<T>(j + 1)]) * (row[pidx<T>(j + 1)] - u);
                if (j > 0) d -= (g[pidx<T>(j - 1)] + gc) * (u - row[pidx<T>(j - 1)]);
                if (line + 1 < m) d += (gc + gd[pidx<T>(j)]) * (dn[pidx<T>(j)] - u);
                if (line > 0) d -= (gu[pidx<T>(j)] + gc) * (u - up[pidx<T>(j)]);
            }
            uout[(int64_t)line * n + j] =
                combine_px<T, ROBUST>(u, num[r], ROBUST ? den[r] : T(0), d, alpha, has_d);
        }
    }
}

// --------------------------------------------------------------------------------------
// stand-alone line convolution (convolver protocol: blur / adjoint / adjoint_pair)

template <typename T>
__global__ void __launch_bounds__(256)
k_conv_lines(ConvLinesArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int n = a.n, m = a.m, TL = a.tl;
    const int P = padded_len<T>(n);
    T *sa = reinterpret_cast<T *>(smem_raw);
    T *stap = sa + TL * P;
    const int64_t fsz = (int64_t)n * m;
    const T *in = static_cast<const T *>(a.in) + blockIdx.y * fsz;
    T *out = static_cast<T *>(a.out) + blockIdx.y * fsz;
    const int l0 = blockIdx.x * TL;
    for (int t = threadIdx.x; t < a.c.ntaps; t += blockDim.x) stap[t] = T(a.taps[t]);
    for (int idx = threadIdx.x; idx < TL * n; idx += blockDim.x) {
        const int li = idx / n, j = idx - li * n;
        if (l0 + li < m) sa[li * P + pidx<T>(j)] = in[(int64_t)(l0 + li) * n + j];
    }
    __syncthreads();
    const int runs = (n + RUN - 1) / RUN;
    for (int q = threadIdx.x; q < TL * runs; q += blockDim.x) {
        const int li = q / runs, j0 = (q - li * runs) * RUN;
        if (l0 + li >= m) continue;
        T v[RUN];
        conv_run<T, true>(sa + li * P, n, j0, a.c, stap, v);
        for (int r = 0; r < RUN && j0 + r < n; ++r) out[(int64_t)(l0 + li) * n + j0 + r] = v[r];
    }
}

// --------------------------------------------------------------------------------------
// batched transpose with optional floor clamp of a second output
// in: [batch][rows][cols] -> out: [batch][cols][rows]

template <typename T>
__global__ void k_transpose(const T *__restrict__ in, T *__restrict__ out, T *__restrict__ out_clamped,
                            int rows, int cols, T floor, int clamp_out) {
    __shared__ T tile[32][33];
    const int64_t fsz = (int64_t)rows * cols;
    in += blockIdx.z * fsz;
    out += blockIdx.z * fsz;
    if (out_clamped) out_clamped += blockIdx.z * fsz;
    const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int r = r0 + i, c = c0 + threadIdx.x;
        if (r < rows && c < cols) tile[i][threadIdx.x] = in[(int64_t)r * cols + c];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int c = c0 + i, r = r0 + threadIdx.x;
        if (r < rows && c < cols) {
            T v = tile[threadIdx.x][i];
            if (out_clamped) out_clamped[(int64_t)c * rows + r] = v > floor ? v : floor;
            if (clamp_out) v = v > floor ? v : floor;
            out[(int64_t)c * rows + r] = v;
        }
    }
}

// elementwise: out = max(in, floor); optional second copy
template <typename T>
__global__ void k_clamp2(const T *__restrict__ in, T *__restrict__ o1, T *__restrict__ o2, int64_t n, T floor) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        T v = in[i];
        v = v > floor ? v : floor;
        o1[i] = v;
        if (o2) o2[i] = v;
    }
}

// --------------------------------------------------------------------------------------
// host-side launchers

template <typename T>
size_t wiener_lines_smem(int n, int lp, int in_vert, bool with_fpos) {
    size_t s = (size_t)lp * fline_stride<sizeof(cx_t<T>)>(n) * sizeof(cx_t<T>);
    if (in_vert && with_fpos) s += (size_t)2 * lp * padded_len<T>(n) * sizeof(T);
    return s;
}

template <typename T>
int wiener_lines_lp(int n) {
    int lp = 2048 / n;
    if (lp > 8) lp = 8;
    if (lp < 1) lp = 1;
    return lp;
}

template <typename T>
cudaError_t launch_wiener_lines(const WienerLinesArgs &a0, int64_t batch, cudaStream_t st) {
    WienerLinesArgs a = a0;
    a.lp = wiener_lines_lp<T>(a.n);
    const size_t smem = wiener_lines_smem<T>(a.n, a.lp, a.in_vert, a.fpos != nullptr);
    cudaError_t e = func_smem_attr((const void *)k_wiener_lines<T>, smem);
    if (e != cudaSuccess) return e;
    const int groups = (a.m + 2 * a.lp - 1) / (2 * a.lp);
    for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
        const int nb = (int)((batch - b0) < 65535 ? (batch - b0) : 65535);
        WienerLinesArgs ab = a;
        const int64_t off = b0 * (int64_t)a.n * a.m * sizeof(T);
        ab.in = static_cast<const char *>(a.in) + off;
        ab.out = static_cast<char *>(a.out) + off;
        if (a.fpos) ab.fpos = static_cast<char *>(a.fpos) + off;
        k_wiener_lines<T><<<dim3(groups, nb), 256, smem, st>>>(ab);
    }
    return cudaGetLastError();
}

template <typename T>
size_t iter_lines_smem(int n, int tl, int ntaps) {
    return ((size_t)(5 * tl + 6) * padded_len<T>(n) + ntaps) * sizeof(T);
}

template <typename T>
int iter_lines_tl(int n) {
    // keep the tile within ~100 KB so two blocks share an SM
    for (int tl = 8; tl >= 1; tl >>= 1)
        if (iter_lines_smem<T>(n, tl, 0) <= 100 * 1024) return tl;
    return 1;
}

template <typename T>
cudaError_t launch_iter_lines(const IterLinesArgs &a0, bool robust, int64_t batch, cudaStream_t st) {
    IterLinesArgs a = a0;
    a.tl = iter_lines_tl<T>(a.n);
    const size_t smem = iter_lines_smem<T>(a.n, a.tl, a.blur.ntaps + a.adj.ntaps);
    auto kern = robust ? k_iter_lines<T, true> : k_iter_lines<T, false>;
    cudaError_t e = func_smem_attr((const void *)kern, smem);
    if (e != cudaSuccess) return e;
    const int tiles = (a.m + a.tl - 1) / a.tl;
    for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
        const int nb = (int)((batch - b0) < 65535 ? (batch - b0) : 65535);
        IterLinesArgs ab = a;
        const int64_t off = b0 * (int64_t)a.n * a.m * sizeof(T);
        ab.u_in = static_cast<const char *>(a.u_in) + off;
        ab.fpos = static_cast<const char *>(a.fpos) + off;
        ab.u_out = static_cast<char *>(a.u_out) + off;
        kern<<<dim3(tiles, nb), 256, smem, st>>>(ab);
    }
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_conv_lines(const ConvLinesArgs &a0, int64_t batch, cudaStream_t st) {
    ConvLinesArgs a = a0;
    a.tl = 8;
    while (a.tl > 1 && ((size_t)a.tl * padded_len<T>(a.n) + a.c.ntaps) * sizeof(T) > 96 * 1024) a.tl >>= 1;
    const size_t smem = ((size_t)a.tl * padded_len<T>(a.n) + a.c.ntaps) * sizeof(T);
    cudaError_t e = func_smem_attr((const void *)k_conv_lines<T>, smem);
    if (e != cudaSuccess) return e;
    const int tiles = (a.m + a.tl - 1) / a.tl;
    for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
        const int nb = (int)((batch - b0) < 65535 ? (batch - b0) : 65535);
        ConvLinesArgs ab = a;
        const int64_t off = b0 * (int64_t)a.n * a.m * sizeof(T);
        ab.in = static_cast<const char *>(a.in) + off;
        ab.out = static_cast<char *>(a.out) + off;
        k_conv_lines<T><<<dim3(tiles, nb), 256, smem, st>>>(ab);
    }
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_transpose(const void *in, void *out, void *out_clamped, int rows, int cols,
                             double floor, int clamp_out, int64_t batch, cudaStream_t st) {
    const int64_t fsz = (int64_t)rows * cols * sizeof(T);
    for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
        const int nb = (int)((batch - b0) < 65535 ? (batch - b0) : 65535);
        dim3 grid((cols + 31) / 32, (rows + 31) / 32, nb);
        k_transpose<T><<<grid, dim3(32, 8), 0, st>>>(
            reinterpret_cast<const T *>(static_cast<const char *>(in) + b0 * fsz),
            reinterpret_cast<T *>(static_cast<char *>(out) + b0 * fsz),
            out_clamped ? reinterpret_cast<T *>(static_cast<char *>(out_clamped) + b0 * fsz) : nullptr,
            rows, cols, T(floor), clamp_out);
    }
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_clamp2(const void *in, void *o1, void *o2, int64_t n, double floor, cudaStream_t st) {
    int blocks = (int)((n + 255) / 256);
    if (blocks > 148 * 16) blocks = 148 * 16;
    k_clamp2<T><<<blocks, 256, 0, st>>>(static_cast<const T *>(in), static_cast<T *>(o1), static_cast<T *>(o2), n, T(floor));
    return cudaGetLastError();
}

// the generic per-iteration line kernel keeps 5 tl + 6 padded lines on chip: it fits while one
// line tile (tl = 1) stays within the opt-in shared memory of a block
bool conv_lines_fits(int dtype, int n, int ntaps) {
    const size_t smem = ((size_t)(dtype == 0 ? padded_len<double>(n) : padded_len<float>(n)) + ntaps) *
                        (dtype == 0 ? 8 : 4);
    return smem <= 227 * 1024;
}

bool iter_lines_fits(int dtype, int n, int ntaps) {
    const size_t smem = dtype == 0 ? iter_lines_smem<double>(n, 1, ntaps) : iter_lines_smem<float>(n, 1, ntaps);
    return smem <= 227 * 1024;
}

#define MD_INST(T)                                                                                 \
    template cudaError_t launch_wiener_lines<T>(const WienerLinesArgs &, int64_t, cudaStream_t);    \
    template cudaError_t launch_iter_lines<T>(const IterLinesArgs &, bool, int64_t, cudaStream_t);  \
    template cudaError_t launch_conv_lines<T>(const ConvLinesArgs &, int64_t, cudaStream_t);        \
    template cudaError_t launch_transpose<T>(const void *, void *, void *, int, int, double, int,   \
                                             int64_t, cudaStream_t);                                \
    template cudaError_t launch_clamp2<T>(const void *, void *, void *, int64_t, double, cudaStream_t);
MD_INST(double)
MD_INST(float)
#undef MD_INST

}  // namespace md
