// md_fused.cu -- placeholder until the cluster-resident iteration kernel lands.
#include "md_fused.h"

namespace md {

bool fused_lines_supported(int, int, int, unsigned) { return false; }

template <typename T> cudaError_t launch_fused_lines(const FusedLinesArgs &, int64_t, cudaStream_t) {
    return cudaErrorNotSupported;
}
template cudaError_t launch_fused_lines<double>(const FusedLinesArgs &, int64_t, cudaStream_t);
template cudaError_t launch_fused_lines<float>(const FusedLinesArgs &, int64_t, cudaStream_t);

}  // namespace md
