// md_lines_fast.h -- interface of the register-window line iteration kernel.
#pragma once

#include <algorithm>
#include <type_traits>

#include "md_internal.h"
#include "md_linefast.cuh"

namespace md {

template <typename T, int R> struct IterFastArgs {
    const T *u_in;
    const T *fpos;
    T *u_out;
    int n, m, periodic;
    DenseTaps<T, R> wb, wa;      // blur / adjoint taps over [-R, R] (kernel parameters)
    T alpha, eps_d2, eps_r2;
    int has_d;
    LutView lut;
};

struct IterFastDesc {
    const void *u_in, *fpos;
    void *u_out;
    int n, m;
    LineConv blur, adj;
    const double *taps_blur_host, *taps_adj_host;   // general taps (host copies), unused for boxes
    double alpha, eps_d2, eps_r2;
    int has_d;
    LutView lut;
};

int line_radius(const LineConv &c);
bool iter_fast_supported(int dtype, int n, const LineConv &blur, const LineConv &adj);
template <typename T> cudaError_t launch_iter_fast(const IterFastDesc &, bool robust, int64_t batch, cudaStream_t);

}  // namespace md
