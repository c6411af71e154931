// md_fused_plane.h -- cluster-resident iteration loop for 2D PSFs (md_fused_plane.cu).
#pragma once

#include <vector>

#include "md_plane_fast.h"

namespace md {

struct FusedPlaneDesc {
    const void *u0, *fpos;    // initial iterate, floored observation
    void *u_out;
    int H, W, periodic, iterations;
    PlaneHalo hb, ha;
    const std::vector<PlaneTap> *taps_blur, *taps_adj;   // host copies
    double alpha, eps_d2, eps_r2;
    int has_d, robust;
    LutView lut;
};

bool fused_plane_supported(int H, int W, const PlaneHalo &hb, const PlaneHalo &ha,
                           const std::vector<PlaneTap> &taps_blur, const std::vector<PlaneTap> &taps_adj, int dtype);
template <typename T> cudaError_t launch_fused_plane(const FusedPlaneDesc &, int64_t batch, cudaStream_t);

}  // namespace md
