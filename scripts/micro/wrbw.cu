// Micro-benchmark: HBM write-only and read-only bandwidth vs copy (B200).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_write(float4* __restrict__ b, long n) {
    const float4 z = make_float4(1.f, 2.f, 3.f, 4.f);
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) b[i] = z;
}
__global__ void k_read(const float4* __restrict__ a, long n, float* sink) {
    float s = 0.f;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        float4 v = __ldcs(&a[i]);
        s += v.x + v.w;
    }
    if (s == 12345.f) *sink = s;
}
__global__ void k_copy(const float4* __restrict__ a, float4* __restrict__ b, long n) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) b[i] = a[i];
}
int main() {
    const long n = (2L << 30) / 16;   // 2 GiB per buffer
    float4 *a, *b;
    float* sink;
    cudaMalloc(&a, n * 16);
    cudaMalloc(&b, n * 16);
    cudaMalloc(&sink, 4);
    cudaMemset(a, 0, n * 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char* name, double bytes, auto launch) {
        launch();
        cudaEventRecord(e0);
        for (int i = 0; i < 10; ++i) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-10s %8.1f GB/s\n", name, bytes * 10 / (ms * 1e-3) / 1e9);
    };
    for (int bpsm : {4, 8, 16}) {
        printf("blocks/SM %d\n", bpsm);
        run("write", n * 16.0, [&] { k_write<<<148 * bpsm, 512>>>(b, n); });
        run("read", n * 16.0, [&] { k_read<<<148 * bpsm, 512>>>(a, n, sink); });
        run("copy", n * 32.0, [&] { k_copy<<<148 * bpsm, 512>>>(a, b, n); });
    }
    return 0;
}
