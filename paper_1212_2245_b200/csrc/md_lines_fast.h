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

// dense tap vector over [-R, R] for one direction of a line convolution
template <typename T, int R>
void fill_dense(DenseTaps<T, R> &d, const LineConv &c, const double *taps_host) {
    for (int k = -R; k <= R; ++k) d.w[k + R] = T(0);
    if (c.kind == LINE_BOX) {
        for (int k = c.lo; k <= c.hi; ++k) d.w[k + R] = T(c.wi);
        if (c.ends) {
            d.w[c.elo + R] = T(c.we);
            d.w[c.ehi + R] = T(c.we);
        }
    } else {
        // out[j] = sum_t w[t] a[j + center - t]  ->  k = center - t
        for (int t = 0; t < c.ntaps; ++t) d.w[c.center - t + R] = T(taps_host[t]);
    }
}
bool iter_fast_supported(int dtype, int n, const LineConv &blur, const LineConv &adj);
template <typename T> cudaError_t launch_iter_fast(const IterFastDesc &, bool robust, int64_t batch, cudaStream_t);

}  // namespace md
