// md_fused64_b.cu -- box specialisations of the float64 cluster kernel for radii 9..16 (split
// from md_fused64.cu to keep compile times short).

#include "md_fused64_kernel.cuh"

namespace md {

cudaError_t launch_fused64_box_hi(const FusedLinesArgs &d, int radius, int64_t batch, cudaStream_t st) {
    switch (radius) {
        case 9: return launch_fused64_box_r<9>(d, batch, st);
        case 10: return launch_fused64_box_r<10>(d, batch, st);
        case 11: return launch_fused64_box_r<11>(d, batch, st);
        case 12: return launch_fused64_box_r<12>(d, batch, st);
        case 13: return launch_fused64_box_r<13>(d, batch, st);
        case 14: return launch_fused64_box_r<14>(d, batch, st);
        case 15: return launch_fused64_box_r<15>(d, batch, st);
        case 16: return launch_fused64_box_r<16>(d, batch, st);
        default: return cudaErrorNotSupported;
    }
}

}  // namespace md
