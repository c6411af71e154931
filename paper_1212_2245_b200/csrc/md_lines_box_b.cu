// md_lines_box_b.cu -- box specialisations of the per-iteration line kernel, radius 9..15
// (md_lines_fast_kernel.cuh; split over two translation units to keep compile times short).
#include "md_lines_fast_kernel.cuh"

namespace md {

template <typename T>
cudaError_t launch_iter_fast_box_b(const IterFastDesc &d, int radius, int64_t batch, cudaStream_t st) {
    switch (radius) {
        case 9: return launch_iter_fast_box_r<T, 9>(d, batch, st);
        case 10: return launch_iter_fast_box_r<T, 10>(d, batch, st);
        case 11: return launch_iter_fast_box_r<T, 11>(d, batch, st);
        case 12: return launch_iter_fast_box_r<T, 12>(d, batch, st);
        case 13: return launch_iter_fast_box_r<T, 13>(d, batch, st);
        case 14: return launch_iter_fast_box_r<T, 14>(d, batch, st);
        case 15: return launch_iter_fast_box_r<T, 15>(d, batch, st);
        default: return cudaErrorInvalidValue;
    }
}

template cudaError_t launch_iter_fast_box_b<double>(const IterFastDesc &, int, int64_t, cudaStream_t);
template cudaError_t launch_iter_fast_box_b<float>(const IterFastDesc &, int, int64_t, cudaStream_t);

}  // namespace md
