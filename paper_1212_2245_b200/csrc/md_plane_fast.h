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
