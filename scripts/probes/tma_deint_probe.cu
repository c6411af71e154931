// Does cuTensorMapEncodeTiled accept the de-interleaving 5D map of md_tma.cuh
// (make_tmap_pairs_deint), and with which strides? Prints the CUresult per variant.
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
int main() {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    void *base = nullptr;
    const long W = 4096, H = 4096;
    cudaMalloc(&base, W * H * 16);
    CUtensorMap m;
    const int hh = 42, rows = 44;
    {
        const cuuint64_t dims[5] = {2, (cuuint64_t)(W / 2), 2, (cuuint64_t)H, 1};
        const cuuint64_t strides[4] = {32, 16, (cuuint64_t)W * 16, (cuuint64_t)(W * H) * 16};
        const cuuint32_t box[5] = {2u, (cuuint32_t)hh, 2u, (cuuint32_t)rows, 1u};
        const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
        CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, base, dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("5D (c, i, e, y, n) strides (32, 16, ...): %d\n", (int)r);
    }
    {   // 4D with the pair as a 16-byte element? (c folded: 2 x f64 as dim0) and dims (c, e, i, y): natural order
        const cuuint64_t dims[5] = {2, 2, (cuuint64_t)(W / 2), (cuuint64_t)H, 1};
        const cuuint64_t strides[4] = {16, 32, (cuuint64_t)W * 16, (cuuint64_t)(W * H) * 16};
        const cuuint32_t box[5] = {2u, 2u, (cuuint32_t)hh, (cuuint32_t)rows, 1u};
        const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
        CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, base, dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("5D natural (c, e, i, y, n): %d\n", (int)r);
    }
    return 0;
}
