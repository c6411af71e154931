// GPC geometry probe: max co-resident clusters per cluster size at one CTA per SM (200 KB
// smem) and two per SM (100 KB), plus which SMs the CTAs of one full wave land on.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int *sm_of) {
    extern __shared__ char s[];
    unsigned smid, cr;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(cr));
    if (threadIdx.x == 0) sm_of[blockIdx.x] = smid;
    s[threadIdx.x] = 1;
}
int main() {
    cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
    printf("SMs %d\n", p.multiProcessorCount);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int per : {1, 2}) {
        size_t smem = per == 1 ? 200 * 1024 : 100 * 1024;
        for (int cs = 1; cs <= 16; ++cs) {
            cudaLaunchConfig_t q = {};
            q.gridDim = dim3(cs); q.blockDim = dim3(256); q.dynamicSmemBytes = smem;
            cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeClusterDimension;
            a[0].val.clusterDim.x = cs; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
            q.attrs = a; q.numAttrs = 1;
            int n = 0; cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &q);
            printf("per_sm %d cluster %2d: max active %3d -> SMs busy %3d (%s)\n", per, cs, n, n * cs / per, cudaGetErrorString(e));
        }
    }
    return 0;
}
