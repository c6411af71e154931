// md_internal.h -- argument blocks shared between the C-ABI layer (md_capi.cu) and the
// kernel translation units. Plain structs passed by value to __global__ functions.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "md_common.cuh"

namespace md {

enum { LINE_BOX = 0, LINE_TAPS = 1 };

// md_last_error() for C-ABI entries outside md_capi.cu; returns `code`
int set_error(int code, const char *msg);

// One direction (blur or adjoint) of a 1D convolution along a line (conv.py:85-173,
// deconv.py:310-326). Box: out[j] = wi * sum_{k=lo..hi} a[j+k] (+ we*(a[j+elo] + a[j+ehi])).
// Taps: out[j] = sum_t w[t] * a[j + center - t]. Indices clamp or wrap.
struct LineConv {
    int kind;
    int periodic;
    int lo, hi, ends, elo, ehi;
    double wi, we;
    int ntaps, center;
};

struct WienerLinesArgs {
    const void *in;       // native frame
    void *out;            // native (out_vert) or line-major
    void *fpos;           // optional line-major max(f, floor)
    int n, log2n, m, lp;
    int in_vert, out_vert, clamp;
    const void *mult;     // Wiener multiplier, bit-reversed order, cx_t<T>[n]
    const void *tw;       // cx_t<T>[n/2]
    double floor;
    int pdl;              // launched as a programmatic dependent of the preceding kernel
};

struct IterLinesArgs {
    const void *u_in;
    const void *fpos;
    void *u_out;
    int n, m, tl;
    LineConv blur, adj;
    const double *taps_blur, *taps_adj;
    double alpha, eps_d2, eps_r2;
    int has_d;
    LutView lut;
};

struct ConvLinesArgs {
    const void *in;
    void *out;
    int n, m, tl;
    LineConv c;
    const double *taps;
};

template <typename T> cudaError_t launch_wiener_lines(const WienerLinesArgs &, int64_t, cudaStream_t);
bool wiener_reg_supported(int dtype, int n);
template <typename T> cudaError_t launch_wiener_reg(const WienerLinesArgs &, int64_t, cudaStream_t);
template <typename T> cudaError_t launch_iter_lines(const IterLinesArgs &, bool robust, int64_t, cudaStream_t);
bool iter_lines_fits(int dtype, int n, int ntaps);
bool conv_lines_fits(int dtype, int n, int ntaps);   // one line of the plain line convolution
template <typename T> cudaError_t launch_conv_lines(const ConvLinesArgs &, int64_t, cudaStream_t);
template <typename T> cudaError_t launch_transpose(const void *in, void *out, void *out_clamped, int rows,
                                                   int cols, double floor, int clamp_out, int64_t batch,
                                                   cudaStream_t);
template <typename T> cudaError_t launch_clamp2(const void *in, void *o1, void *o2, int64_t n, double floor,
                                                cudaStream_t);

}  // namespace md
