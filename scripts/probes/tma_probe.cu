// TMA 3D box loads of float / double fields (md_tma.cuh helpers): which shapes work?
// nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I paper_1212_2245_b200/csrc scripts/probes/tma_probe.cu -o /tmp/tma_probe
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "md_tma.cuh"
using namespace md;
template <typename T>
__global__ void k(const __grid_constant__ CUtensorMap m, T *out, int bw, int bh, int x, int y) {
    extern __shared__ __align__(128) unsigned char sm[];
    T *s = reinterpret_cast<T *>(sm);
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + ((bw * bh * sizeof(T) + 7) & ~size_t(7)));
    if (threadIdx.x == 0) {
        tma_bar_arm(bar, bw * bh * sizeof(T));
        tma_load_3d(s, &m, x, y, 0, bar);
    }
    __syncthreads();
    tma_bar_wait(bar);
    for (int i = threadIdx.x; i < bw * bh; i += blockDim.x) out[i] = s[i];
}
template <typename T>
void run(int W, int H, int bw, int bh, int x, int y) {
    std::vector<T> h(W * H);
    for (int i = 0; i < W * H; ++i) h[i] = (T)(i + 1);
    T *d, *o;
    cudaMalloc(&d, W * H * sizeof(T));
    cudaMalloc(&o, bw * bh * sizeof(T));
    cudaMemcpy(d, h.data(), W * H * sizeof(T), cudaMemcpyHostToDevice);
    CUtensorMap m{};
    bool ok = make_tmap_3d(&m, d, sizeof(T), W, H, 1, bw, bh);
    size_t sm = bw * bh * sizeof(T) + 16;
    cudaFuncSetAttribute(k<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k<T><<<1, 128, sm>>>(m, o, bw, bh, x, y);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<T> r(bw * bh);
    int bad = 0;
    if (e == cudaSuccess) {
        cudaMemcpy(r.data(), o, r.size() * sizeof(T), cudaMemcpyDeviceToHost);
        for (int j = 0; j < bh; ++j)
            for (int i = 0; i < bw; ++i) {
                int gx = x + i, gy = y + j;
                T want = (gx >= 0 && gx < W && gy >= 0 && gy < H) ? h[gy * W + gx] : T(0);
                bad += r[j * bw + i] != want;
            }
    }
    printf("%s W=%d H=%d box %dx%d at (%d,%d): map %d, %s, %d wrong\n", sizeof(T) == 8 ? "f64" : "f32", W, H, bw, bh, x, y, ok,
           cudaGetErrorString(e), bad);
    if (e != cudaSuccess) { cudaDeviceReset(); }
    cudaFree(d); cudaFree(o);
}
int main(int argc, char **argv) {
    // one case per process: tma_probe.bin f64|f32 W H bw bh x y
    const bool dbl = argv[1][1] == '6';
    const int W = atoi(argv[2]), H = atoi(argv[3]), bw = atoi(argv[4]), bh = atoi(argv[5]), x = atoi(argv[6]), y = atoi(argv[7]);
    if (dbl) run<double>(W, H, bw, bh, x, y);
    else run<float>(W, H, bw, bh, x, y);
    return 0;
}
