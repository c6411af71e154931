// Probe: a persistent "filler" kernel of N CTAs, each holding `smem` bytes of shared memory (so it
// cannot share an SM with a 182 KB cluster-kernel CTA) and spinning for `ns` nanoseconds; records
// the SM each CTA ran on. Used to test whether work launched next to the float64 cluster kernel
// lands only on the SMs whole-GPC cluster placement leaves idle.
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k_filler(int *smid_out, long long ns) {
    extern __shared__ char s[];
    unsigned id;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(id));
    if (threadIdx.x == 0) smid_out[blockIdx.x] = (int)id;
    long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    long long t = t0;
    while (t - t0 < ns) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    s[threadIdx.x] = (char)t;
}
extern "C" int launch_filler(void *stream, int ctas, int smem, long long ns, int *smid_out) {
    cudaFuncSetAttribute(k_filler, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_filler<<<ctas, 256, smem, (cudaStream_t)stream>>>(smid_out, ns);
    return (int)cudaGetLastError();
}
