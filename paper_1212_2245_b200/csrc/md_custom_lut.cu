// md_custom_lut.cu -- DivergenceLut with NON-default parameters (deconv.py:81-139: any
// 0 < delta < direct_below < upper and step), and the plan-free pointwise steps a
// caller-supplied convolver object needs (the ratio f / b (x W) and _combine, deconv.py:421-446).
//
// The default table is compiled into the pipeline kernels (md_common.cuh constants); a custom
// one lives in a device array built here and is evaluated with runtime parameters, in the
// reference's rounding order (NumPy's separate array operations, no FMA contraction).

#include <cmath>

#include "md_internal.h"
#include "md_plane.h"

namespace md {

struct CustomLut {
    const double *t;
    int64_t count;
    double delta, inv_step, upper, direct_below, slope, intercept;
};

// xs = delta + step * arange(count); table = xs - 1 - ln xs (deconv.py:101-112)
__global__ void k_lut_build_custom(double *t, int64_t count, double delta, double step) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        const double x = __dadd_rn(__dmul_rn(step, (double)i), delta);
        t[i] = __dsub_rn(__dsub_rn(x, 1.0), log(x));
    }
}

// DivergenceLut.r1 (deconv.py:114-134), runtime parameters
__device__ __forceinline__ double r1_custom(const CustomLut &L, double x) {
    double pos = __dmul_rn(__dsub_rn(x < L.upper ? x : L.upper, L.delta), L.inv_step);
    long long idx = (long long)pos;
    idx = idx < 0 ? 0 : (idx > L.count - 2 ? L.count - 2 : idx);
    pos = __dsub_rn(pos, (double)idx);
    const double lo = L.t[idx], hi = L.t[idx + 1];
    double r = __dadd_rn(__dmul_rn(__dsub_rn(hi, lo), pos), lo);
    if (x > L.upper) r = __dadd_rn(__dmul_rn(L.slope, x), L.intercept);
    if (x < L.direct_below) r = __dsub_rn(__dsub_rn(x, 1.0), log(x));
    return r;
}

__global__ void k_lut_r1_custom(CustomLut L, const double *__restrict__ x, double *__restrict__ out, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = r1_custom(L, x[i]);
}

// _weight_arrays (deconv.py:142-162) with a custom table: r = r1(b / fsafe) fsafe, the
// small-observation limit max(b - f, 0) below the floor, W = 0.5 / sqrt(r + eps^2)
template <typename T>
__global__ void k_robust_weight_custom(CustomLut L, const T *__restrict__ f, const T *__restrict__ b,
                                       T *__restrict__ out, int64_t n, double eps2, double floor, int floored) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double fv = (double)f[i], bv = (double)b[i];
        const bool small = !floored && fv < floor;
        const double fs = small ? 1.0 : fv;
        double r = __dmul_rn(r1_custom(L, __ddiv_rn(bv, fs)), fs);
        if (small) r = bv - fv > 0.0 ? bv - fv : 0.0;
        r = __dadd_rn(r, eps2);
        out[i] = (T)__ddiv_rn(0.5, __dsqrt_rn(r));
    }
}

static int ew_grid(int64_t n) { return (int)std::min<int64_t>((n + 255) / 256, 148 * 16); }

}  // namespace md

using namespace md;

#include "../../include/mdcuda.h"

extern "C" {

static CustomLut make_lut(const double *table, int64_t count, double delta, double step, double upper,
                          double direct_below, double slope, double intercept) {
    CustomLut L;
    L.t = table; L.count = count; L.delta = delta; L.inv_step = 1.0 / step; L.upper = upper;
    L.direct_below = direct_below; L.slope = slope; L.intercept = intercept;
    return L;
}

static bool lut_args_ok(const double *table, int64_t count, double delta, double step, double upper,
                        double direct_below) {
    return table && count >= 2 && step > 0.0 && 0.0 < delta && delta < direct_below && direct_below < upper;
}

int32_t md_lut_build(double *table, int64_t count, double delta, double step, void *stream) {
    if (!table || count < 2 || !(step > 0.0) || !(delta > 0.0)) return set_error(-1, "bad table arguments");
    k_lut_build_custom<<<ew_grid(count), 256, 0, static_cast<cudaStream_t>(stream)>>>(table, count, delta, step);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : set_error(-3, cudaGetErrorString(e));
}

int32_t md_lut_r1_custom(const double *table, int64_t count, double delta, double step, double upper,
                         double direct_below, double slope, double intercept, const double *x, double *out,
                         int64_t n, void *stream) {
    if (!lut_args_ok(table, count, delta, step, upper, direct_below) || !x || !out || n < 0)
        return set_error(-1, "bad arguments");
    if (n == 0) return 0;
    const CustomLut L = make_lut(table, count, delta, step, upper, direct_below, slope, intercept);
    k_lut_r1_custom<<<ew_grid(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(L, x, out, n);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : set_error(-3, cudaGetErrorString(e));
}

int32_t md_robust_weight_custom(int32_t dtype, const double *table, int64_t count, double delta, double step,
                                double upper, double direct_below, double slope, double intercept, const void *f,
                                const void *b, void *out, int64_t n, double eps_data, double floor,
                                int32_t assume_floored, void *stream) {
    if (!lut_args_ok(table, count, delta, step, upper, direct_below) || !f || !b || !out || n < 0 ||
        (dtype != 0 && dtype != 1))
        return set_error(-1, "bad arguments");
    if (n == 0) return 0;
    const CustomLut L = make_lut(table, count, delta, step, upper, direct_below, slope, intercept);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (dtype == 0)
        k_robust_weight_custom<double><<<ew_grid(n), 256, 0, st>>>(L, static_cast<const double *>(f),
                                                                   static_cast<const double *>(b),
                                                                   static_cast<double *>(out), n,
                                                                   eps_data * eps_data, floor, assume_floored);
    else
        k_robust_weight_custom<float><<<ew_grid(n), 256, 0, st>>>(L, static_cast<const float *>(f),
                                                                  static_cast<const float *>(b),
                                                                  static_cast<float *>(out), n,
                                                                  eps_data * eps_data, floor, assume_floored);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : set_error(-3, cudaGetErrorString(e));
}

int32_t md_ratio(int32_t dtype, const void *f, const void *b, const void *w, void *out, int64_t n, void *stream) {
    if (!f || !b || !out || n < 0 || (dtype != 0 && dtype != 1)) return set_error(-1, "bad arguments");
    if (n == 0) return 0;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const cudaError_t e = dtype == 0 ? launch_ratio<double>(f, b, w, out, n, st) : launch_ratio<float>(f, b, w, out, n, st);
    return e == cudaSuccess ? 0 : set_error(-3, cudaGetErrorString(e));
}

int32_t md_clamp(int32_t dtype, const void *in, void *out, int64_t n, double floor, void *stream) {
    if (!in || !out || n < 0 || (dtype != 0 && dtype != 1)) return set_error(-1, "bad arguments");
    if (n == 0) return 0;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const cudaError_t e = dtype == 0 ? launch_clamp2<double>(in, out, nullptr, n, floor, st)
                                     : launch_clamp2<float>(in, out, nullptr, n, floor, st);
    return e == cudaSuccess ? 0 : set_error(-3, cudaGetErrorString(e));
}

int32_t md_combine(int32_t dtype, const void *u, const void *num, const void *den, const void *d, void *out,
                   int64_t n, double alpha, void *stream) {
    if (!u || !num || !out || n < 0 || (dtype != 0 && dtype != 1)) return set_error(-1, "bad arguments");
    if (n == 0) return 0;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const cudaError_t e = dtype == 0 ? launch_combine<double>(u, num, den, d, out, n, d ? alpha : 0.0, st)
                                     : launch_combine<float>(u, num, den, d, out, n, d ? alpha : 0.0, st);
    return e == cudaSuccess ? 0 : set_error(-3, cudaGetErrorString(e));
}

}  // extern "C"
