// md_lines_box_a.cu -- box specialisations of the per-iteration line kernel, radius 1..8
// (md_lines_fast_kernel.cuh; split over two translation units to keep compile times short).
#include "md_lines_fast_kernel.cuh"

namespace md {

template <typename T>
cudaError_t launch_iter_fast_box_a(const IterFastDesc &d, int radius, int64_t batch, cudaStream_t st) {
    switch (radius) {
        case 1: return launch_iter_fast_box_r<T, 1>(d, batch, st);
        case 2: return launch_iter_fast_box_r<T, 2>(d, batch, st);
        case 3: return launch_iter_fast_box_r<T, 3>(d, batch, st);
        case 4: return launch_iter_fast_box_r<T, 4>(d, batch, st);
        case 5: return launch_iter_fast_box_r<T, 5>(d, batch, st);
        case 6: return launch_iter_fast_box_r<T, 6>(d, batch, st);
        case 7: return launch_iter_fast_box_r<T, 7>(d, batch, st);
        case 8: return launch_iter_fast_box_r<T, 8>(d, batch, st);
        default: return cudaErrorInvalidValue;
    }
}

template cudaError_t launch_iter_fast_box_a<double>(const IterFastDesc &, int, int64_t, cudaStream_t);
template cudaError_t launch_iter_fast_box_a<float>(const IterFastDesc &, int, int64_t, cudaStream_t);

}  // namespace md
