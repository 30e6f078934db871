// Micro-benchmark: HBM bandwidth of a 2-D strided copy with contiguous segments of
// SEG bytes (the access shape of the strided FFT passes), vs. a contiguous copy.
#include <cstdio>
#include <cuda_runtime.h>
template <int SEGF2>   // segment length in float2
__global__ void k_seg(const float2* __restrict__ a, float2* __restrict__ b, int rows, int nx) {
    // tile = SEGF2 columns x 512 rows, threads walk rows
    const int tiles_x = nx / SEGF2;
    const int tile = blockIdx.x;
    const int xt = tile % tiles_x, rg = tile / tiles_x;
    const int q = threadIdx.x % SEGF2, r0 = threadIdx.x / SEGF2;
    const int rstep = blockDim.x / SEGF2;
    for (int r = r0; r < 512; r += rstep) {
        const long idx = ((long)rg * 512 + r) * nx + (long)xt * SEGF2 + q;
        b[idx] = a[idx];
    }
}
__global__ void k_flat(const float4* __restrict__ a, float4* __restrict__ b, long n) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) b[i] = a[i];
}
int main() {
    const int nx = 1024;
    const long rows = 512L * 256;           // 1 GiB of float2 per buffer
    const long n = rows * nx;
    float2 *a, *b;
    cudaMalloc(&a, n * 8);
    cudaMalloc(&b, n * 8);
    cudaMemset(a, 0, n * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char* name, auto launch) {
        launch();
        cudaEventRecord(e0);
        for (int i = 0; i < 10; ++i) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-12s %8.1f GB/s\n", name, 2.0 * n * 8 * 10 / (ms * 1e-3) / 1e9);
    };
    run("flat16B", [&] { k_flat<<<148 * 8, 512>>>((const float4*)a, (float4*)b, n / 2); });
    const int tiles = (int)(rows / 512) * 0;   // unused
    (void)tiles;
    run("seg32B", [&] { k_seg<4><<<(int)(rows / 512) * (nx / 4), 256>>>(a, b, (int)rows, nx); });
    run("seg64B", [&] { k_seg<8><<<(int)(rows / 512) * (nx / 8), 256>>>(a, b, (int)rows, nx); });
    run("seg128B", [&] { k_seg<16><<<(int)(rows / 512) * (nx / 16), 256>>>(a, b, (int)rows, nx); });
    run("seg256B", [&] { k_seg<32><<<(int)(rows / 512) * (nx / 32), 256>>>(a, b, (int)rows, nx); });
    run("seg512B", [&] { k_seg<64><<<(int)(rows / 512) * (nx / 64), 256>>>(a, b, (int)rows, nx); });
    return 0;
}
