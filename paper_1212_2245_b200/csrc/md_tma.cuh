// md_tma.cuh -- tensor-memory-accelerator (TMA) tile loads for the plane stage kernels.
//
// A tile of a [N][H][W] field (row-major frames) is one cp.async.bulk.tensor.3d copy into
// dense shared rows, completed on an mbarrier as a transaction count: no per-element address
// arithmetic, no register round trip, and the positions outside the field arrive as zeros (the
// tensor map's out-of-bounds fill), which is exactly the zero halo stage B's u tile needs.
// The tensor maps are encoded on the host per launch (cuTensorMapEncodeTiled, reached through
// the runtime's driver entry point: no libcuda link) and passed as __grid_constant__ kernel
// parameters.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>

namespace md {

// ------------------------------------------------------------------------------ device side
__device__ __forceinline__ uint32_t tma_smem(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t smem_addr_of(const void *p) { return tma_smem(p); }

// one-thread setup of a single-use barrier: init (one arrival), make it visible to the async
// proxy, arm it with the bytes of the copies that will complete on it
__device__ __forceinline__ void tma_bar_arm(uint64_t *bar, uint32_t bytes) {
    const uint32_t b = tma_smem(bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
}

// box at (x, y, z) of the map into shared memory (dst 128-byte aligned), completing on bar
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, int x, int y, int z, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            tma_smem(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(tma_smem(bar))
        : "memory");
}

// every thread: wait for phase 0 of the barrier (the copies have landed and are visible)
__device__ __forceinline__ void tma_bar_wait(uint64_t *bar) {
    const uint32_t b = tma_smem(bar);
    uint32_t done;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(b)
            : "memory");
    } while (!done);
}

// ------------------------------------------------------------------------------ host side
// A [n][h][w] field of `esz`-byte elements, boxes of box_w x box_h x 1. False (no map) when the
// TMA constraints are not met: 16-byte aligned base, row pitch a multiple of 16 bytes, box
// rows a multiple of 16 bytes, box sides <= 256 -- the caller then keeps the per-element path.
inline bool make_tmap_3d(CUtensorMap *map, const void *base, size_t esz, int64_t w, int64_t h, int64_t n, int box_w,
                         int box_h) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    if (!encode || (reinterpret_cast<uintptr_t>(base) & 15) || ((size_t)w * esz) % 16 || ((size_t)box_w * esz) % 16 ||
        box_w < 1 || box_w > 256 || box_h < 1 || box_h > 256 || w < 1 || h < 1 || n < 1)
        return false;
    const cuuint64_t dims[3] = {(cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)n};
    const cuuint64_t strides[2] = {(cuuint64_t)w * esz, (cuuint64_t)w * h * esz};
    const cuuint32_t box[3] = {(cuuint32_t)box_w, (cuuint32_t)box_h, 1u};
    const cuuint32_t estr[3] = {1u, 1u, 1u};
    const CUtensorMapDataType dt = esz == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    return encode(map, dt, 3, const_cast<void *>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace md
