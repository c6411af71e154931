// md_fused_box_b -- box specialisations of the fused kernel, radius 9..15 (split over two
// translation units to keep compile times short).
#include "md_fused_kernel.cuh"

namespace md {

template <typename T>
cudaError_t launch_fused_box_partb(const FusedLinesArgs &d, int radius, int64_t batch, cudaStream_t st) {
    switch (radius) {
        case 9: return launch_fused_box_lpw<T, 9>(d, batch, st);
        case 10: return launch_fused_box_lpw<T, 10>(d, batch, st);
        case 11: return launch_fused_box_lpw<T, 11>(d, batch, st);
        case 12: return launch_fused_box_lpw<T, 12>(d, batch, st);
        case 13: return launch_fused_box_lpw<T, 13>(d, batch, st);
        case 14: return launch_fused_box_lpw<T, 14>(d, batch, st);
        case 15: return launch_fused_box_lpw<T, 15>(d, batch, st);
        default: return cudaErrorInvalidValue;
    }
}

template cudaError_t launch_fused_box_partb<double>(const FusedLinesArgs &, int, int64_t, cudaStream_t);
template cudaError_t launch_fused_box_partb<float>(const FusedLinesArgs &, int, int64_t, cudaStream_t);

}  // namespace md
