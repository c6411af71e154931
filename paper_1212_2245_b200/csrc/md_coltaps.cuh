// md_coltaps.cuh -- 2D tap lists regrouped by column for register reuse between two output
// rows (direct 2D convolution of _SpatialConvolver / _FourierConvolver2D, deconv.py:295-376).
//
// A column is a fixed dx with a run of consecutive dy (interior gaps get zero weights).
// Walking a column downwards from its first tap, loaded value i feeds the upper output row
// with tap i and the lower row with tap i - 1, so a row pair costs len + 1 shared-memory
// loads per column instead of 2 len; the FMAs stay 2 len. Direct 2D convolution is bound by
// the shared-memory pipe, so this is the lever (measured 1.25x on the 2D cluster kernel).
#pragma once

#include <map>
#include <vector>

#include "md_plane.h"

namespace md {

constexpr int kColMax = 64;          // columns
constexpr int kColWeights = 256;     // weights over all column runs

template <typename T> struct Vec2;
template <> struct Vec2<float> { using type = float2; };
template <> struct Vec2<double> { using type = double2; };

// c[k].x = dy0 * stride + dx (offset of the column's first tap), c[k].y = len | (first weight << 16)
template <typename T> struct ColTaps {
    int ncol;
    int2 c[kColMax];
    T w[kColWeights];
};

// host: taps -> columns for a shared-memory row stride; false if the limits are exceeded
// (ct == nullptr: only check)
template <typename T>
inline bool build_col_taps(const std::vector<PlaneTap> &taps, int stride, ColTaps<T> *ct) {
    std::map<int, std::map<int, double>> by_dx;
    for (const PlaneTap &t : taps) by_dx[t.dx][t.dy] += t.w;
    if (by_dx.size() > (size_t)kColMax) return false;
    int nw = 0, nc = 0;
    for (const auto &col : by_dx) {
        const int dy0 = col.second.begin()->first, dy1 = col.second.rbegin()->first;
        const int len = dy1 - dy0 + 1;
        if (nw + len > kColWeights) return false;
        if (ct) {
            ct->c[nc] = make_int2(dy0 * stride + col.first, len | (nw << 16));
            for (int i = 0; i < len; ++i) {
                const auto it = col.second.find(dy0 + i);
                ct->w[nw + i] = it == col.second.end() ? T(0) : T(it->second);
            }
        }
        nw += len;
        ++nc;
    }
    if (ct) ct->ncol = nc;
    return true;
}

// convolution of a row pair: a0 = upper row, a1 = lower row; s points at the upper row's first
// output column; J outputs per row at column stride XS
template <typename T, int J, int XS>
__device__ __forceinline__ void col_taps_pair(const T *s, int rs, const ColTaps<T> &tp, T a0[J], T a1[J]) {
#pragma unroll
    for (int j = 0; j < J; ++j) a0[j] = a1[j] = T(0);
    for (int c = 0; c < tp.ncol; ++c) {
        const int2 ci = tp.c[c];
        const T *p = s + ci.x;
        const int len = ci.y & 0xffff;
        const T *wc = tp.w + (ci.y >> 16);
        T wp = wc[0];
#pragma unroll
        for (int j = 0; j < J; ++j) a0[j] += wp * p[XS * j];
        for (int i = 1; i < len; ++i) {
            p += rs;
            const T wi = wc[i];
#pragma unroll
            for (int j = 0; j < J; ++j) {
                const T v = p[XS * j];
                a0[j] += wi * v;
                a1[j] += wp * v;
            }
            wp = wi;
        }
        p += rs;
#pragma unroll
        for (int j = 0; j < J; ++j) a1[j] += wp * p[XS * j];
    }
}

// adjoint pair of a row pair over interleaved (p, W): n = sum w p, d = sum w W
template <typename T, int J, int XS>
__device__ __forceinline__ void col_taps_pair2(const typename Vec2<T>::type *s, int rs, const ColTaps<T> &tp,
                                               T n0[J], T n1[J], T d0[J], T d1[J]) {
    using T2 = typename Vec2<T>::type;
#pragma unroll
    for (int j = 0; j < J; ++j) n0[j] = n1[j] = d0[j] = d1[j] = T(0);
    for (int c = 0; c < tp.ncol; ++c) {
        const int2 ci = tp.c[c];
        const T2 *p = s + ci.x;
        const int len = ci.y & 0xffff;
        const T *wc = tp.w + (ci.y >> 16);
        T wp = wc[0];
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const T2 v = p[XS * j];
            n0[j] += wp * v.x;
            d0[j] += wp * v.y;
        }
        for (int i = 1; i < len; ++i) {
            p += rs;
            const T wi = wc[i];
#pragma unroll
            for (int j = 0; j < J; ++j) {
                const T2 v = p[XS * j];
                n0[j] += wi * v.x;
                d0[j] += wi * v.y;
                n1[j] += wp * v.x;
                d1[j] += wp * v.y;
            }
            wp = wi;
        }
        p += rs;
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const T2 v = p[XS * j];
            n1[j] += wp * v.x;
            d1[j] += wp * v.y;
        }
    }
}

}  // namespace md
