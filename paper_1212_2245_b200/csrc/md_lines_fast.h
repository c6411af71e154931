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
    T box_wi;                    // box specialisation (BOXR > 0): interior weight
    T alpha_w, guard_w, one_w;   // alpha, the division guard and 1 divided by box_wi
    T box_cb[4], box_ca[4];      // weight corrections at k = -R, -R+1, R-1, R (blur, adjoint)
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
// host: a box line convolution as interior weight wi over [-R, R] plus corrections at
// k = -R, -R+1, R-1, R; false when it has no such form (then the dense path runs)
template <typename T, int R>
bool box_corrections(const LineConv &c, double wi, T corr[4]) {
    DenseTaps<T, R> d;
    fill_dense<T, R>(d, c, nullptr);
    for (int k = -R + 2; k <= R - 2; ++k)
        if (d.w[k + R] != T(wi)) return false;
    if (R == 1) {                                    // k = -R+1 = R-1 = 0: must be interior
        if (d.w[1] != T(wi)) return false;
        corr[0] = d.w[0] - T(wi); corr[1] = corr[2] = T(0); corr[3] = d.w[2] - T(wi);
        return true;
    }
    const int ks[4] = {-R, -R + 1, R - 1, R};
    for (int i = 0; i < 4; ++i) corr[i] = d.w[ks[i] + R] - T(wi);
    return true;
}

bool iter_fast_supported(int dtype, int n, const LineConv &blur, const LineConv &adj);
template <typename T> cudaError_t launch_iter_fast(const IterFastDesc &, bool robust, int64_t batch, cudaStream_t);
// box blur / adjoint of radius 1..15 as O(1) sliding sums (md_lines_box_a/b.cu); returns
// cudaErrorNotSupported when the kernels have no such form (the dense path then runs)
template <typename T> cudaError_t launch_iter_fast_box_a(const IterFastDesc &, int radius, int64_t, cudaStream_t);
template <typename T> cudaError_t launch_iter_fast_box_b(const IterFastDesc &, int radius, int64_t, cudaStream_t);

}  // namespace md
