// md_wiener_fast.cu -- per-line Wiener filter with a register-resident four-step FFT.
//
// Replaces apply_column_filter(a, conj(h)/(|h|^2+K)) (fft.py:236-258, deconv.py:253-254,
// 666-672) for line lengths n = S*S (S = 8, 16, 32). Two lines ride in one complex
// transform (real / imaginary part, as in the reference). For j = j1 + S*j2 and
// k = k2 + S*k1:
//   forward  : thread j1: S-point DFT over j2 (registers) -> x W_n^{j1 k2} -> smem transpose
//              thread k2: S-point DFT over j1 (registers) -> X[k2 + S k1]
//   filter   : X *= M[k]                                    (registers)
//   inverse  : thread k2: inverse DFT over k1 -> x W_n^{-j1 k2} -> smem transpose
//              thread j1: inverse DFT over k2 -> x'[j1 + S j2] / n
// so a line pair costs two shared-memory transposes and no global round trip.
#include "md_internal.h"

namespace md {

// cos / sin of 2*pi*k/32, k = 0..31 (compile-time twiddles for S <= 32)
__device__ constexpr double kC32[32] = {
    1.0, 0.98078528040323043, 0.92387953251128674, 0.83146961230254524, 0.70710678118654757,
    0.55557023301960218, 0.38268343236508978, 0.19509032201612825, 0.0, -0.19509032201612825,
    -0.38268343236508978, -0.55557023301960218, -0.70710678118654757, -0.83146961230254524,
    -0.92387953251128674, -0.98078528040323043, -1.0, -0.98078528040323043, -0.92387953251128674,
    -0.83146961230254524, -0.70710678118654757, -0.55557023301960218, -0.38268343236508978,
    -0.19509032201612825, 0.0, 0.19509032201612825, 0.38268343236508978, 0.55557023301960218,
    0.70710678118654757, 0.83146961230254524, 0.92387953251128674, 0.98078528040323043};

template <int S> __host__ __device__ constexpr int bitrev(int x) {
    int r = 0;
    for (int b = 1; b < S; b <<= 1) {
        r = (r << 1) | (x & 1);
        x >>= 1;
    }
    return r;
}

// in-register S-point transforms, in place, all indices compile-time:
//   dif_reg : natural order in, bit-reversed order out, forward twiddles exp(-2 pi i k / 2h)
//   dit_reg : bit-reversed order in, natural order out, inverse (conjugate) twiddles, unscaled
template <typename T>
__device__ __forceinline__ cx_t<T> twmul(cx_t<T> b, int k, int half, bool inv) {
    if (k == 0) return b;
    if (4 * k == 2 * half) return inv ? mkc<T>(-b.y, b.x) : mkc<T>(b.y, -b.x);   // -+ i
    const int ti = k * (32 / (2 * half));
    const T c = T(kC32[ti]);
    const T sn = T(kC32[(ti + 24) & 31]);          // sin(2 pi ti / 32)
    const T s = inv ? sn : -sn;
    return mkc<T>(b.x * c - b.y * s, b.x * s + b.y * c);
}

template <typename T, int S>
__device__ __forceinline__ void dif_reg(cx_t<T> (&v)[S]) {
#pragma unroll
    for (int half = S / 2; half >= 1; half >>= 1) {
#pragma unroll
        for (int g = 0; g < S; g += 2 * half) {
#pragma unroll
            for (int k = 0; k < half; ++k) {
                const cx_t<T> a = v[g + k], b = v[g + k + half];
                v[g + k] = cadd(a, b);
                v[g + k + half] = twmul<T>(csub(a, b), k, half, false);
            }
        }
    }
}

template <typename T, int S>
__device__ __forceinline__ void dit_inv_reg(cx_t<T> (&v)[S]) {
#pragma unroll
    for (int half = 1; half < S; half <<= 1) {
#pragma unroll
        for (int g = 0; g < S; g += 2 * half) {
#pragma unroll
            for (int k = 0; k < half; ++k) {
                const cx_t<T> t = twmul<T>(v[g + k + half], k, half, true);
                const cx_t<T> a = v[g + k];
                v[g + k + half] = csub(a, t);
                v[g + k] = cadd(a, t);
            }
        }
    }
}

template <typename T, int S>
__global__ void __launch_bounds__(256, S <= 16 ? (sizeof(T) == 4 ? 3 : 2) : 1)   // float 3 blocks/SM (<= 85 regs), double 2
k_wiener_lines_reg(WienerLinesArgs a) {
    // programmatic dependent launch (md_capi.cu, run_lines_pipelined): this grid may start while
    // the preceding cluster iteration kernel still runs; its last block waits for that kernel
    // to finish, so this grid's completion implies the predecessor's
    if (a.pdl && blockIdx.x == gridDim.x - 1 && blockIdx.y == gridDim.y - 1)
        asm volatile("griddepcontrol.wait;\n" ::: "memory");
    using C = cx_t<T>;
    constexpr int N = S * S;
    constexpr int PB = 256 / S;                 // line pairs per block
    constexpr int TS = S + 1;                   // transpose row stride (padding)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *tw = reinterpret_cast<C *>(smem_raw);    // W_n^(q k) at [k][q], q, k < S
    C *tr = tw + N;                             // PB transposes of S x TS
    const int m = a.m;
    const int64_t fr = blockIdx.y;
    const int64_t fsz = (int64_t)N * m;
    const T *in = static_cast<const T *>(a.in) + fr * fsz;
    T *out = static_cast<T *>(a.out) + fr * fsz;
    T *fpos = a.fpos ? static_cast<T *>(a.fpos) + fr * fsz : nullptr;
    const T floor = T(a.floor);
    const C *twg = static_cast<const C *>(a.tw);
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        // inter-step twiddles arranged [k][q] = W_n^(q k) (q, k < S, q k < n): the lanes of a
        // step read consecutive entries (a W_n^(q k) lookup by q k strides the banks for even k)
        const int k = (i / S) * (i % S);
        const C t = twg[k & (N / 2 - 1)];         // the plan table holds W_n^k for k < n/2
        tw[i] = k < N / 2 ? t : mkc<T>(-t.x, -t.y);
    }
    const int t = threadIdx.x;
    // thread -> (pair p, lane-in-pair q); vertical input: p fastest for coalescing
    const int p = a.in_vert ? t % PB : t / S;
    const int q = a.in_vert ? t / PB : t % S;
    const int pair = blockIdx.x * PB + p;
    const int l0 = 2 * pair, l1 = 2 * pair + 1;
    const bool v0 = l0 < m, v1 = l1 < m;
    C *T2 = tr + p * (S * TS + 1);             // +1: spread pairs over banks

    // ---- load x[q + S j2] (q = j1), fpos
    C v[S];
#pragma unroll
    for (int j2 = 0; j2 < S; ++j2) {
        const int j = q + S * j2;
        T x0 = T(0), x1 = T(0);
        if (a.in_vert) {
            if (v0) x0 = in[(int64_t)j * m + l0];
            if (v1) x1 = in[(int64_t)j * m + l1];
        } else {
            if (v0) x0 = in[(int64_t)l0 * N + j];
            if (v1) x1 = in[(int64_t)l1 * N + j];
        }
        v[j2] = mkc<T>(x0, x1);
    }
    // fpos after ALL loads: a store between them (possible alias of `in`) would serialise the
    // loads behind each other's latency
    if (fpos && !a.in_vert) {
#pragma unroll
        for (int j2 = 0; j2 < S; ++j2) {
            const int j = q + S * j2;
            if (v0) fpos[(int64_t)l0 * N + j] = v[j2].x > floor ? v[j2].x : floor;
            if (v1) fpos[(int64_t)l1 * N + j] = v[j2].y > floor ? v[j2].y : floor;
        }
    }
    constexpr int NP = N + 1;
    const int lbase = 2 * blockIdx.x * PB;
    if (fpos && a.in_vert) {
        // vertical input: fpos line-major from the loaded registers, staged through the (still
        // free) transpose buffer so that consecutive threads store consecutive samples of a line
        T *st = reinterpret_cast<T *>(tr);
#pragma unroll
        for (int j2 = 0; j2 < S; ++j2) {
            const int j = q + S * j2;
            st[(2 * p) * NP + j] = v[j2].x > floor ? v[j2].x : floor;
            st[(2 * p + 1) * NP + j] = v[j2].y > floor ? v[j2].y : floor;
        }
        __syncthreads();
        for (int idx = threadIdx.x; idx < 2 * PB * N; idx += blockDim.x) {
            const int li = idx / N, j = idx - li * N;
            if (lbase + li < m) fpos[(int64_t)(lbase + li) * N + j] = st[li * NP + j];
        }
    }
    __syncthreads();                            // twiddle table ready (and the staging read)
    // ---- forward: DFT over j2 (X[k2] lands at v[rev(k2)]), twiddle W_n^{j1 k2}, transpose
    dif_reg<T, S>(v);
#pragma unroll
    for (int k2 = 0; k2 < S; ++k2) T2[k2 * TS + q] = cmul(v[bitrev<S>(k2)], tw[k2 * S + q]);
    __syncthreads();
    // thread q = k2 now: DFT over j1 (X[k2 + S k1] lands at v[rev(k1)])
#pragma unroll
    for (int j1 = 0; j1 < S; ++j1) v[j1] = T2[q * TS + j1];
    dif_reg<T, S>(v);
    // ---- filter X[k2 + S k1] *= M (M stored in natural order for this kernel)
    const C *mult = static_cast<const C *>(a.mult);
#pragma unroll
    for (int k1 = 0; k1 < S; ++k1) v[bitrev<S>(k1)] = cmul(v[bitrev<S>(k1)], __ldg(mult + q + S * k1));
    // ---- inverse: DFT^-1 over k1 (bit-reversed in, natural j1 out), twiddle W_n^{-j1 k2}
    dit_inv_reg<T, S>(v);
#pragma unroll
    for (int j1 = 0; j1 < S; ++j1) T2[q * TS + j1] = cmulc(v[j1], tw[j1 * S + q]);
    __syncthreads();
#pragma unroll
    for (int k2 = 0; k2 < S; ++k2) v[bitrev<S>(k2)] = T2[k2 * TS + q];
    dit_inv_reg<T, S>(v);
    const T inv_n = T(1) / T(N);
    // ---- store x'[q + S j2]
    if (!a.in_vert && !a.out_vert) {
#pragma unroll
        for (int j2 = 0; j2 < S; ++j2) {
            const int j = q + S * j2;
            T y0 = v[j2].x * inv_n, y1 = v[j2].y * inv_n;
            if (a.clamp) { y0 = y0 > floor ? y0 : floor; y1 = y1 > floor ? y1 : floor; }
            if (v0) out[(int64_t)l0 * N + j] = y0;
            if (v1) out[(int64_t)l1 * N + j] = y1;
        }
        return;
    }
    if (a.in_vert && a.out_vert) {
#pragma unroll
        for (int j2 = 0; j2 < S; ++j2) {
            const int j = q + S * j2;
            T y0 = v[j2].x * inv_n, y1 = v[j2].y * inv_n;
            if (a.clamp) { y0 = y0 > floor ? y0 : floor; y1 = y1 > floor ? y1 : floor; }
            if (v0) out[(int64_t)j * m + l0] = y0;
            if (v1) out[(int64_t)j * m + l1] = y1;
        }
        return;
    }
    // vertical input -> line-major output (and fpos): stage the pair through shared memory so
    // that consecutive threads write consecutive samples of a line. Staged lines are NP = N + 1
    // apart: the column-order writes (consecutive threads = consecutive lines) then hit distinct
    // banks instead of one (a stride of N words is a multiple of 32)
    __syncthreads();
    T *st = reinterpret_cast<T *>(tr);          // 2 PB lines x NP reals (fits: PB (S TS + 1) complex)
#pragma unroll
    for (int j2 = 0; j2 < S; ++j2) {
        const int j = q + S * j2;
        T y0 = v[j2].x * inv_n, y1 = v[j2].y * inv_n;
        if (a.clamp) { y0 = y0 > floor ? y0 : floor; y1 = y1 > floor ? y1 : floor; }
        st[(2 * p) * NP + j] = y0;
        st[(2 * p + 1) * NP + j] = y1;
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < 2 * PB * N; idx += blockDim.x) {
        const int li = idx / N, j = idx - li * N;
        if (lbase + li < m) out[(int64_t)(lbase + li) * N + j] = st[li * NP + j];
    }
}

static_assert(2 * 16 * (256 + 1) <= 2 * 16 * (16 * 17 + 1), "staging fits the transpose buffer (S = 16)");

template <typename T, int S>
cudaError_t launch_wiener_reg_t(const WienerLinesArgs &a, int64_t batch, cudaStream_t st) {
    constexpr int PB = 256 / S;
    const size_t smem = (size_t)(S * S + PB * (S * (S + 1) + 1)) * sizeof(cx_t<T>);
    cudaError_t e = func_smem_attr((const void *)k_wiener_lines_reg<T, S>, smem);
    if (e != cudaSuccess) return e;
    const int groups = (a.m + 2 * PB - 1) / (2 * PB);
    const int64_t fb = (int64_t)a.n * a.m * sizeof(T);
    for (int64_t b0 = 0; b0 < batch; b0 += 65535) {
        const int nb = (int)((batch - b0) < 65535 ? (batch - b0) : 65535);
        WienerLinesArgs ab = a;
        ab.in = static_cast<const char *>(a.in) + b0 * fb;
        ab.out = static_cast<char *>(a.out) + b0 * fb;
        if (a.fpos) ab.fpos = static_cast<char *>(a.fpos) + b0 * fb;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(groups, nb);
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = (a.pdl && b0 == 0) ? 1 : 0;
        ab.pdl = a.pdl && b0 == 0;
        e = cudaLaunchKernelEx(&cfg, k_wiener_lines_reg<T, S>, ab);
        if (e != cudaSuccess) return e;
    }
    return cudaGetLastError();
}

bool wiener_reg_supported(int dtype, int n) {
    if (n == 64 || n == 256) return true;
    return n == 1024 && dtype == 1;              // 32 complex registers per thread: float only
}

template <typename T>
cudaError_t launch_wiener_reg(const WienerLinesArgs &a, int64_t batch, cudaStream_t st) {
    if (a.n == 64) return launch_wiener_reg_t<T, 8>(a, batch, st);
    if (a.n == 256) return launch_wiener_reg_t<T, 16>(a, batch, st);
    return launch_wiener_reg_t<T, 32>(a, batch, st);
}

template cudaError_t launch_wiener_reg<double>(const WienerLinesArgs &, int64_t, cudaStream_t);
template cudaError_t launch_wiener_reg<float>(const WienerLinesArgs &, int64_t, cudaStream_t);

}  // namespace md
