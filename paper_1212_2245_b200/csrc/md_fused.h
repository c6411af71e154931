// md_fused.h -- the cluster-resident whole-iteration-loop kernel for 1D blur on small frames.
#pragma once

#include "md_internal.h"

namespace md {

struct FusedLinesArgs {
    const void *u_in;      // line-major u0 (clamped Wiener)
    const void *fpos;      // line-major max(f, floor)
    void *u_out;           // native-layout result
    int n, m, iterations, out_vert;
    LineConv blur, adj;
    const double *taps_blur_host, *taps_adj_host;
    double alpha, eps_d2, eps_r2;
    int has_d, robust;
    LutView lut;
    int *query;            // non-null: store the resident cluster count, launch nothing
    int *query_geom;       // with query: [cluster CTAs, CTAs per SM] of that launch (optional)
    int floor_f;           // float64 kernel: `fpos` is the raw line-major observation, floored in the
    double floor;          // kernel (max(f, floor) exactly as the Wiener epilogue: no fpos field)
};

// radius: max(blur, adjoint) line radius (line_radius, md_lines_fast.h)
bool fused_lines_supported(int dtype, int n, int m, unsigned flags, int radius);
int fused_lpw(int dtype, int radius);
template <typename T> cudaError_t launch_fused_box_parta(const FusedLinesArgs &, int radius, int64_t, cudaStream_t);
template <typename T> cudaError_t launch_fused_box_partb(const FusedLinesArgs &, int radius, int64_t, cudaStream_t);
template <typename T>
inline cudaError_t launch_fused_box(const FusedLinesArgs &d, int radius, int64_t batch, cudaStream_t st) {
    return radius <= 8 ? launch_fused_box_parta<T>(d, radius, batch, st) : launch_fused_box_partb<T>(d, radius, batch, st);
}
template <typename T> cudaError_t launch_fused_lines(const FusedLinesArgs &, int64_t batch, cudaStream_t);
// float64, radius <= 8: the shuffle-window / st.async-halo kernel (md_fused64.cu);
// cudaErrorNotSupported when it does not apply
cudaError_t launch_fused64(const FusedLinesArgs &, int64_t batch, cudaStream_t);
int fused64_rows();   // lines per CTA of that kernel

}  // namespace md
