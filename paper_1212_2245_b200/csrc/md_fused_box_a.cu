// md_fused_box_a -- box specialisations of the fused kernel, radius 1..8 (split over two
// translation units to keep compile times short).
#include "md_fused_kernel.cuh"

namespace md {

template <typename T>
cudaError_t launch_fused_box_parta(const FusedLinesArgs &d, int radius, int64_t batch, cudaStream_t st) {
    switch (radius) {
        case 1: return launch_fused_box_lpw<T, 1>(d, batch, st);
        case 2: return launch_fused_box_lpw<T, 2>(d, batch, st);
        case 3: return launch_fused_box_lpw<T, 3>(d, batch, st);
        case 4: return launch_fused_box_lpw<T, 4>(d, batch, st);
        case 5: return launch_fused_box_lpw<T, 5>(d, batch, st);
        case 6: return launch_fused_box_lpw<T, 6>(d, batch, st);
        case 7: return launch_fused_box_lpw<T, 7>(d, batch, st);
        case 8: return launch_fused_box_lpw<T, 8>(d, batch, st);
        default: return cudaErrorInvalidValue;
    }
}

template cudaError_t launch_fused_box_parta<double>(const FusedLinesArgs &, int, int64_t, cudaStream_t);
template cudaError_t launch_fused_box_parta<float>(const FusedLinesArgs &, int, int64_t, cudaStream_t);

}  // namespace md
