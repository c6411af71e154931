// md_plane_fast.h -- interface of the register-blocked 2D direct-tap iteration stages.
#pragma once

#include <vector>

#include "md_coltaps.cuh"

namespace md {

constexpr int kPlaneMaxTaps = 128;

template <typename T> struct PlaneFastArgs {
    const T *u, *f;     // iterate, floored observation
    T *p, *w, *u_out;
    int H, W, periodic;
    int slab, gy0, Hg;  // slab mode: rows read directly (halo present); global row of row 0; global height
    int ylo, yhi;       // slab mode: rows [ylo, yhi) of the buffers exist (relative to the base pointers);
                        // tile rows outside only feed discarded outputs and read the nearest valid row
    PlaneHalo hb, ha;
    int ssa, ssb;       // shared row strides of the stage-A u tile and the stage-B (p, W) tile
    ColTaps<T> tb, ta;  // column-grouped taps for those strides
    T alpha, eps_d2, eps_r2;
    int has_d;
    LutView lut;
    int tma_a, tma_b;   // the u tiles come by TMA (md_tma.cuh): stage A's interior tiles, all of stage B's
    int pwi;            // p and W interleaved as pairs in the p buffer (2 elements per pixel; w unused)
    int tma_pw;         // ... and stage B's interior (p, W) tiles come by TMA
    int pw_split;       // ... stored parity-split per row (even columns, then odd: k_plane_b_adj)
};

// Stage B with two ADJACENT output columns per thread (float64): the (p, W) pair tile is stored
// de-interleaved by column parity ([parity][row][column pair]: stage A writes the pair field
// parity-split per row, so each half is one plain TMA box), and a lane's input column 2l + e sits
// at l + (e >> 1) of half (e & 1) -- consecutive across lanes, conflict-free for any tap offset.
// A merged column d walks the union of the dy-runs of tap columns d (for output 2l) and d - 1
// (for output 2l + 1): each loaded pair feeds up to 8 outputs (4 rows x 2 columns)
// instead of 4. Weights outside a tap column's run are zero (an FMA of +0 leaves the sum bitwise
// unchanged), so every output still sums its taps in the column-walk order: results are the
// same bit for bit.
constexpr int kAdjColMax = 72;
constexpr int kAdjWeights = 320;
template <typename T> struct AdjTaps {
    int ncol;
    int hle, hh;                            // tile starts at x0 - hle (hle even >= hl); hh pairs per half row
    int2 c[kAdjColMax];                     // .x = tile offset (half * rows * hh + lo * hh + col), .y = len | (w0 << 16)
    typename Vec2<T>::type w[kAdjWeights];  // (weight for output 2l, weight for output 2l + 1) per step
};

struct PlaneFastDesc {
    const void *u, *f;
    void *p, *w, *u_out;
    int H, W, periodic;
    int slab, gy0, Hg;         // see PlaneFastArgs
    int a_begin, a_end;        // slab: stage A computes rows [a_begin, a_end) (relative to own row 0;
                               // the full stage is [-adj.ht, H + adj.hb)); empty = skipped
    int b_begin, b_end;        // slab: stage B computes own rows [b_begin, b_end) (full: [0, H))
    int halo_top, halo_bot;    // slab: rows present above / below the own rows in every buffer
    PlaneHalo hb, ha;
    const std::vector<PlaneTap> *taps_blur, *taps_adj;   // host copies
    double alpha, eps_d2, eps_r2;
    int has_d;
    LutView lut;
    int pw_pairs;              // whole-frame launches: p / W interleaved in the p buffer (2 elements per pixel)
};

bool plane_fast_supported(const PlaneHalo &hb, const PlaneHalo &ha, const std::vector<PlaneTap> &taps_blur,
                          const std::vector<PlaneTap> &taps_adj, int dtype);
template <typename T> cudaError_t launch_plane_fast(const PlaneFastDesc &, bool robust, int64_t, cudaStream_t);

}  // namespace md
