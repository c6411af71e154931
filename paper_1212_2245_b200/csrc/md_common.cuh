// md_common.cuh -- shared device helpers: complex arithmetic, the divergence table r1,
// the robust weight and the TV diffusivity. Templated on the arithmetic type T
// (double for parity-critical configs, float where measured parity allows).
#pragma once

#include <cuda_runtime.h>
#include <cstdio>
#include <stdint.h>

#include <map>
#include <mutex>
#include <utility>

namespace md {

// ---- checked build (-DMD_CHECKED; scripts/build_checked.sh): device-side bounds and protocol
// assertions in the cluster kernels plus NaN-poisoned shared memory, the substitute for
// compute-sanitizer (closed on this pool). Compiled out of the production library.
#ifdef MD_CHECKED
#define MD_CHECK(cond)                                                                                  \
    do {                                                                                                \
        if (!(cond)) {                                                                                  \
            printf("MD_CHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__,          \
                   (int)blockIdx.x, (int)threadIdx.x);                                                  \
            __trap();                                                                                   \
        }                                                                                               \
    } while (0)
#else
#define MD_CHECK(cond) \
    do {               \
    } while (0)
#endif

// bytes of dynamic shared memory this launch has (PTX %dynamic_smem_size)
__device__ __forceinline__ uint32_t dyn_smem_bytes() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(r));
    return r;
}
// checked build: fill this CTA's dynamic shared memory with NaN bytes before first use, so a
// read of a never-written element that reaches a result turns the result into NaN
__device__ __forceinline__ void poison_smem(unsigned char *smem) {
#ifdef MD_CHECKED
    const uint32_t n = dyn_smem_bytes();
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) smem[i] = 0xff;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // before TMA writes the same bytes
    __syncthreads();
#else
    (void)smem;
#endif
}

// host: raise a kernel's dynamic shared-memory limit (and allow non-portable cluster sizes)
// once per (kernel, device), not on every launch -- cudaFuncSetAttribute costs microseconds,
// which batch-1 latency notices. The attribute is one value per function, so the limit only
// ever grows (to the largest size any caller launched with); thread-safe.
inline cudaError_t func_smem_attr(const void *kern, size_t smem, bool nonportable_cluster = false) {
    struct State { size_t smem = 0; bool nonportable = false; };
    static std::mutex mu;
    static std::map<std::pair<const void *, int>, State> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    State &st = done[std::make_pair(kern, dev)];
    if (smem > st.smem) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        st.smem = smem;
    }
    if (nonportable_cluster && !st.nonportable) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
        st.nonportable = true;
    }
    return cudaSuccess;
}

template <typename T> struct Cx;
template <> struct Cx<double> { using type = double2; };
template <> struct Cx<float> { using type = float2; };
template <typename T> using cx_t = typename Cx<T>::type;

template <typename C> __device__ __forceinline__ C cmul(C a, C b) {
    C r; r.x = a.x * b.x - a.y * b.y; r.y = a.x * b.y + a.y * b.x; return r;
}
// a * conj(b)
template <typename C> __device__ __forceinline__ C cmulc(C a, C b) {
    C r; r.x = a.x * b.x + a.y * b.y; r.y = a.y * b.x - a.x * b.y; return r;
}
template <typename C> __device__ __forceinline__ C cadd(C a, C b) { C r; r.x = a.x + b.x; r.y = a.y + b.y; return r; }
template <typename C> __device__ __forceinline__ C csub(C a, C b) { C r; r.x = a.x - b.x; r.y = a.y - b.y; return r; }
template <typename C> __device__ __forceinline__ C cscale(C a, decltype(a.x) s) { C r; r.x = a.x * s; r.y = a.y * s; return r; }
template <typename T> __device__ __forceinline__ cx_t<T> mkc(T re, T im) { cx_t<T> r; r.x = re; r.y = im; return r; }

// --------------------------------------------------------------------------------------
// divergence table r1(s) = s - 1 - ln s, deconv.py:81-139. The table itself lives in global
// memory (133,057 entries, built on the device at plan time by k_build_lut); these are the
// evaluation rules of DivergenceLut.r1 (deconv.py:114-134).
constexpr double kLutDelta = 1.0 / 32.0;
constexpr double kLutInvStep = 2048.0;
constexpr double kLutUpper = 65.0;
constexpr double kLutDirectBelow = 0.5;
constexpr int kLutCount = 133057;                 // round((65 - 1/32) * 2048) + 1
// linear continuation above `upper`, matching value and slope of x - 1 - ln x at 65
// (deconv.py:108-112, 127-129): slope 1 - 1/65, intercept (65 - 1 - ln 65) - slope * 65
constexpr double kLutSlope = 64.0 / 65.0;
constexpr double kLutIntercept = -4.1743872698956395;   // as the reference rounds it

struct LutView {
    const double *t64;
    const float *t32;
    const float2 *p32;                            // (t32[i], t[i+1] - t[i]), i < kLutCount - 1
    const double2 *p64;                           // (t[i], t[i+1] - t[i]) in float64, i < kLutCount - 1
};

__device__ __forceinline__ double lut_fetch(const LutView &L, int i, double) { return __ldg(L.t64 + i); }
__device__ __forceinline__ float lut_fetch(const LutView &L, int i, float) { return __ldg(L.t32 + i); }
__device__ __forceinline__ double dlog(double x) { return log(x); }
__device__ __forceinline__ float dlog(float x) { return __logf(x); }
__device__ __forceinline__ double drsqrt(double x) { return rsqrt(x); }
__device__ __forceinline__ float drsqrt(float x) { return rsqrtf(x); }

template <typename T>
__device__ __forceinline__ T r1_lut(const LutView &L, T x) {
    if (x < T(kLutDirectBelow)) return x - T(1) - dlog(x);
    if (x > T(kLutUpper)) return T(kLutSlope) * x + T(kLutIntercept);
    T pos = (x - T(kLutDelta)) * T(kLutInvStep);
    int i = (int)pos;                              // pos >= (0.5 - 1/32) * 2048 > 0 here
    i = i > kLutCount - 2 ? kLutCount - 2 : i;
    T t = pos - T(i);
    T lo = lut_fetch(L, i, T(0));
    T hi = lut_fetch(L, i + 1, T(0));
    return lo + (hi - lo) * t;
}

// W = 0.5 / sqrt(fpos * r1(b / fpos) + eps_d^2) for a floored observation (deconv.py:142-162)
template <typename T>
__device__ __forceinline__ T robust_weight_floored(const LutView &L, T fpos, T b, T eps2) {
    T r = r1_lut(L, b / fpos) * fpos;
    return T(0.5) / sqrt(r + eps2);
}

// general form: observations below `floor` use max(b - f, 0) (deconv.py:147-158)
template <typename T>
__device__ __forceinline__ T robust_weight_general(const LutView &L, T f, T b, T eps2, T floor) {
    T r;
    if (f < floor) r = b - f > T(0) ? b - f : T(0);
    else r = r1_lut(L, b / f) * f;
    return T(0.5) / sqrt(r + eps2);
}

constexpr double kGuard = 1e-12;                   // DIVISION_GUARD, deconv.py:74

// u' = (u * num) / max(den, guard) with the alpha split of D (deconv.py:421-446)
template <typename T, bool ROBUST>
__device__ __forceinline__ T combine_px(T u, T num, T den, T d, T alpha, bool has_d) {
    if (has_d) {
        num += alpha * (d > T(0) ? d : T(0));
        T neg = alpha * (d < T(0) ? d : T(0));
        den = ROBUST ? den - neg : T(1) - neg;
    } else if (!ROBUST) {
        return u * num;
    }
    den = den > T(kGuard) ? den : T(kGuard);
    return (u * num) / den;
}

}  // namespace md
