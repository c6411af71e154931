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

// R output rows per thread (the pair kernels above are R = 2): walking a column of len taps
// from its first tap, loaded value i feeds output row r with tap i - r (0 <= i - r < len), so
// R rows cost len + R - 1 loads per column instead of R (len + 1) / 2 -- each row's sum still
// runs over the same taps in the same order (columns in turn, taps top to bottom), so the
// results equal the pair kernels' bit for bit. The head (i < R - 1) and tail (i >= len) steps,
// where only some rows take part, are unrolled; the middle steps feed all R rows. The R
// weights of a step are a register window shifted by one table read per step.
// V: the loaded element (T, or Vec2<T> for the adjoint pair); F(acc_row, w, v): the update
template <typename T, typename V, int R, int J, int XS, bool SHORT, typename Acc, typename F>
__device__ __forceinline__ void col_walk_one(const V *p, int rs, const T *wc, int len, Acc (&acc)[R][J], F upd) {
    // SHORT = false: len >= R - 1, so every head step is a tap of its rows and every tail step
    // lies past the head -- no per-step predicates (the common case); SHORT: any len
    T w[R];                                       // w[r] = wc[i - r] at step i
#pragma unroll
    for (int r = 0; r < R; ++r) w[r] = T(0);
    // head: steps 0 .. R-2 (rows 0 .. i)
#pragma unroll
    for (int i = 0; i < R - 1; ++i) {
#pragma unroll
        for (int r = R - 1; r > 0; --r) w[r] = w[r - 1];
        w[0] = (!SHORT || i < len) ? wc[i] : T(0);
        V v[J];
#pragma unroll
        for (int j = 0; j < J; ++j) v[j] = p[XS * j];
#pragma unroll
        for (int r = 0; r <= i; ++r)
            if (!SHORT || i - r < len) {
#pragma unroll
                for (int j = 0; j < J; ++j) upd(acc[r][j], w[r], v[j]);
            }
        p += rs;
    }
    // middle: steps R-1 .. len-1, every row
    for (int i = R - 1; i < len; ++i) {
#pragma unroll
        for (int r = R - 1; r > 0; --r) w[r] = w[r - 1];
        w[0] = wc[i];
        V v[J];
#pragma unroll
        for (int j = 0; j < J; ++j) v[j] = p[XS * j];
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int j = 0; j < J; ++j) upd(acc[r][j], w[r], v[j]);
        p += rs;
    }
    // tail: steps i = len + t (t = 0 .. R-2) not already taken by the head; rows t+1 .. R-1
    // (and r <= i). When len < R - 1 the pointer already stands at step R - 1.
#pragma unroll
    for (int t = 0; t < R - 1; ++t) {
        const int i = len + t;
        if (SHORT && i < R - 1) continue;
#pragma unroll
        for (int r = R - 1; r > 0; --r) w[r] = w[r - 1];
        w[0] = T(0);
        V v[J];
#pragma unroll
        for (int j = 0; j < J; ++j) v[j] = p[XS * j];
#pragma unroll
        for (int r = t + 1; r < R; ++r)
            if (!SHORT || r <= i) {
#pragma unroll
                for (int j = 0; j < J; ++j) upd(acc[r][j], w[r], v[j]);
            }
        p += rs;
    }
}

// a column of exactly LEN taps, fully unrolled: no loop, no predicates; the LEN weights are
// read once (uniform registers) -- the common short columns of line / small 2D PSFs
template <typename T, typename V, int R, int J, int XS, int LEN, typename Acc, typename F>
__device__ __forceinline__ void col_walk_fixed(const V *p, int rs, const T *wc, Acc (&acc)[R][J], F upd) {
    T w[LEN];
#pragma unroll
    for (int k = 0; k < LEN; ++k) w[k] = wc[k];
#pragma unroll
    for (int i = 0; i < LEN + R - 1; ++i) {
        V v[J];
#pragma unroll
        for (int j = 0; j < J; ++j) v[j] = p[XS * j];
#pragma unroll
        for (int r = 0; r < R; ++r)
            if (i - r >= 0 && i - r < LEN) {
#pragma unroll
                for (int j = 0; j < J; ++j) upd(acc[r][j], w[i - r], v[j]);
            }
        p += rs;
    }
}

#ifndef MD_COL_FIXED
#define MD_COL_FIXED 1              // columns of up to 8 taps take the unrolled walk (0: never)
#endif
template <typename T, typename V, int R, int J, int XS, typename Acc, typename F>
__device__ __forceinline__ void col_walk_rows(const V *s, int rs, const ColTaps<T> &tp, Acc (&acc)[R][J], F upd) {
    for (int c = 0; c < tp.ncol; ++c) {
        const int2 ci = tp.c[c];
        const int len = ci.y & 0xffff;
        const T *wc = tp.w + (ci.y >> 16);
        // the branches are uniform (every thread walks the same column); a switch, so the
        // length selects its walk through one indexed branch instead of a compare chain
        const V *p = s + ci.x;
        switch (MD_COL_FIXED ? len : 0) {
            case 1: col_walk_fixed<T, V, R, J, XS, 1>(p, rs, wc, acc, upd); break;
            case 2: col_walk_fixed<T, V, R, J, XS, 2>(p, rs, wc, acc, upd); break;
            case 3: col_walk_fixed<T, V, R, J, XS, 3>(p, rs, wc, acc, upd); break;
            case 4: col_walk_fixed<T, V, R, J, XS, 4>(p, rs, wc, acc, upd); break;
            case 5: col_walk_fixed<T, V, R, J, XS, 5>(p, rs, wc, acc, upd); break;
            case 6: col_walk_fixed<T, V, R, J, XS, 6>(p, rs, wc, acc, upd); break;
            case 7: col_walk_fixed<T, V, R, J, XS, 7>(p, rs, wc, acc, upd); break;
            case 8: col_walk_fixed<T, V, R, J, XS, 8>(p, rs, wc, acc, upd); break;
            default:
                if (len >= R - 1) col_walk_one<T, V, R, J, XS, false>(p, rs, wc, len, acc, upd);
                else col_walk_one<T, V, R, J, XS, true>(p, rs, wc, len, acc, upd);
        }
    }
}

// blur of R rows: a[r][j] = sum w u
template <typename T, int R, int J, int XS>
__device__ __forceinline__ void col_taps_rows(const T *s, int rs, const ColTaps<T> &tp, T (&a)[R][J]) {
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
        for (int j = 0; j < J; ++j) a[r][j] = T(0);
    col_walk_rows<T, T, R, J, XS>(s, rs, tp, a, [](T &acc, T w, T v) { acc += w * v; });
}

// adjoint pair of R rows over interleaved (p, W): nd[r][j].x = sum w p, .y = sum w W
template <typename T, int R, int J, int XS>
__device__ __forceinline__ void col_taps_rows2(const typename Vec2<T>::type *s, int rs, const ColTaps<T> &tp,
                                               typename Vec2<T>::type (&nd)[R][J]) {
    using T2 = typename Vec2<T>::type;
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
        for (int j = 0; j < J; ++j) nd[r][j].x = nd[r][j].y = T(0);
    col_walk_rows<T, T2, R, J, XS>(s, rs, tp, nd, [](T2 &acc, T w, T2 v) {
        acc.x += w * v.x;
        acc.y += w * v.y;
    });
}

}  // namespace md
