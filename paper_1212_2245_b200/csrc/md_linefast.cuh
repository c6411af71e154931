// md_linefast.cuh -- register-window building blocks for line (1D blur) kernels.
//
// A warp owns whole lines; lane s holds the 8 consecutive samples j = 8s .. 8s+7 of a line
// ("segment"). Lines live in shared memory extended by a halo of HW samples on each side
// (edge-replicated for the clamped convolvers, wrapped for the periodic ones) in a
// "9-stride" layout -- one pad word after every 8 samples -- so that the 32 lanes of a warp,
// whose segments start 8 samples apart, hit 32 distinct banks, and so that every element of
// a lane's window sits at a COMPILE-TIME offset from the lane's base address. Convolutions
// then need no index arithmetic at all: out[r] = sum_k w[k] * v[r + k], k in [-R, R], with
// the dense tap vector w passed as kernel parameters (constant-bank FFMA operands).
#pragma once

#include "md_common.cuh"

namespace md {

constexpr int SEG = 8;

template <int R> struct HaloOf { static constexpr int value = R <= 8 ? 8 : (R <= 16 ? 16 : 32); };

// storage index of extended sample e (0 <= e < n + 2*HW)
__host__ __device__ constexpr int xaddr(int e) { return e + (e >> 3); }
__host__ __device__ constexpr int xline_len(int n, int hw) { return xaddr(n + 2 * hw) + 1; }

// compile-time offset of element k (relative to the segment start) from the lane base
__host__ __device__ constexpr int koff(int k) { return k + (k >= 0 ? k / 8 : -((-k + 7) / 8)); }

template <typename T, int R> struct DenseTaps { T w[2 * R + 1]; };

// window convolution of 8 outputs: dense taps over [-R, R] (constant-bank FMAs), or, for a
// box (equal interior weights) of radius BOXR (= R), an O(1)-per-output sliding sum over
// [-R, R] plus weight corrections at k = -R, -R+1, R-1, R (even-length and fractional boxes:
// deconv.py box convolver, conv.py:141-173). SCALE = false (plain integer boxes only) leaves
// the window sums unscaled by the interior weight, for callers that fold 1/wi elsewhere.
template <typename T, int R, int BOXR, bool BOXC, bool SCALE = true>
__device__ __forceinline__ void conv_window(const T (&v)[SEG + 2 * R], const DenseTaps<T, R> &taps, T box_wi,
                                            const T (&corr)[4], T out[SEG]) {
    if constexpr (BOXR > 0) {
        static_assert(BOXR == R, "box window radius must equal the register window radius");
        // short dependency chains (few warps per scheduler): the first window by a pairwise
        // tree, then the running sum over precomputed entering-minus-leaving differences
        T t[2 * R + 1];
#pragma unroll
        for (int i = 0; i <= 2 * R; ++i) t[i] = v[i];
#pragma unroll
        for (int w = 1; w <= 2 * R; w *= 2)
#pragma unroll
            for (int i = 0; i + w <= 2 * R; i += 2 * w) t[i] += t[i + w];
        T d[SEG];
#pragma unroll
        for (int r = 1; r < SEG; ++r) d[r] = v[r + 2 * R] - v[r - 1];
        static_assert(SCALE || !BOXC, "unscaled windows only for plain boxes");
        T s = t[0];
        out[0] = SCALE ? s * box_wi : s;
#pragma unroll
        for (int r = 1; r < SEG; ++r) {
            s += d[r];
            out[r] = SCALE ? s * box_wi : s;
        }
        if constexpr (BOXC) {
#pragma unroll
            for (int r = 0; r < SEG; ++r)
                out[r] += corr[0] * v[r] + corr[1] * v[r + 1] + corr[2] * v[r + 2 * R - 1] + corr[3] * v[r + 2 * R];
        }
    } else {
#pragma unroll
        for (int r = 0; r < SEG; ++r) {
            T acc = T(0);
#pragma unroll
            for (int k = -R; k <= R; ++k) acc += taps.w[k + R] * v[r + k + R];
            out[r] = acc;
        }
    }
}


// fast reciprocal / reciprocal square root / log: one MUFU op for float (operands here are
// positive normal numbers: b >= 1e-12, fpos >= floor, q + eps^2 > 0), Newton-refined for double
__device__ __forceinline__ float frcp(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
// double: the MUFU estimate y0 (about 2^-22 relative) corrected by the cubic series of the
// residual e = 1 - x y0: 1 / x = y0 / (1 - e) = y0 (1 + e + e^2 + O(e^3)), i.e.
// fma(y0, fma(e, e, e), y0) -- three dependent DFMAs instead of two Newton steps' four, and
// within an ulp or two of the IEEE quotient (the dropped e^3 term is ~2^-66; operands here are
// positive normal numbers, so no special-case path)
__device__ __forceinline__ double frcp(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double e = fma(-x, y, 1.0);
    return fma(y, fma(e, e, e), y);
}
__device__ __forceinline__ float frsqrt(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
// double: residual e = 1 - x y0^2 of the MUFU estimate, then (1 - e)^(-1/2) = 1 + e/2 + 3e^2/8
// + O(e^3): y0 + y0 e (1/2 + 3e/8) -- five DP operations instead of two Newton steps' seven
__device__ __forceinline__ double frsqrt(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double e = fma(-x, y * y, 1.0);
    return fma(y, e * fma(e, 0.375, 0.5), y);
}
__device__ __forceinline__ float flog(float x) {
    float r;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r * 0.69314718055994531f;
}
__device__ __forceinline__ double flog(double x) { return log(x); }

// max(x, y) as one compare and a select (x > y ? x : y): the reference's guards and D+ parts
// (np.maximum) on ordinary numbers. fmax() and the same ternary in C compile to a min/max
// compare plus NaN / signed-zero fix-ups (4-5 instructions per double); the operands here are
// finite, and where they compare equal (+-0 against 0) the sign of a zero never reaches a result
__device__ __forceinline__ double dmax_sel(double x, double y) {
    double r;
    asm("{\n\t.reg .pred p;\n\tsetp.gt.f64 p, %1, %2;\n\tselp.f64 %0, %1, %2, p;\n\t}" : "=d"(r) : "d"(x), "d"(y));
    return r;
}
__device__ __forceinline__ float dmax_sel(float x, float y) { return x > y ? x : y; }
__device__ __forceinline__ double dmin_sel(double x, double y) {
    double r;
    asm("{\n\t.reg .pred p;\n\tsetp.lt.f64 p, %1, %2;\n\tselp.f64 %0, %1, %2, p;\n\t}" : "=d"(r) : "d"(x), "d"(y));
    return r;
}
__device__ __forceinline__ float dmin_sel(float x, float y) { return x < y ? x : y; }

__device__ __forceinline__ float lut_interp(const LutView &L, int i, float t) {
    const float2 p = __ldg(L.p32 + i);            // one 8-byte load: value and step
    return p.x + p.y * t;
}
__device__ __forceinline__ double lut_interp(const LutView &L, int i, double t) {
    const double lo = __ldg(L.t64 + i), hi = __ldg(L.t64 + i + 1);
    return lo + (hi - lo) * t;
}

// r1 by table interpolation with both extensions evaluated branch-free (deconv.py:114-134);
// a warp-vote skip of the rare direct-formula branch measured slower (reconvergence)
template <typename T>
__device__ __forceinline__ T r1_fast(const LutView &L, T x) {
    const T xc = x < T(kLutUpper) ? x : T(kLutUpper);
    T pos = (xc - T(kLutDelta)) * T(kLutInvStep);
    pos = pos > T(0) ? pos : T(0);
    int i = (int)pos;
    i = i < kLutCount - 2 ? i : kLutCount - 2;
    T r = lut_interp(L, i, pos - T(i));
    if (x > T(kLutUpper)) r = T(kLutSlope) * x + T(kLutIntercept);
    if (x < T(kLutDirectBelow)) r = x - T(1) - flog(x);
    return r;
}

}  // namespace md
