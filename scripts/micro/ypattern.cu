// Micro-benchmark: HBM bandwidth of the strided y-pass pattern (tiles of Q consecutive kx x
// L rows of one plane, row stride Nx) -- pass B reads Ky rows and writes 2 Ky rows, pass D the
// reverse -- and of pass C's plane-stride pattern split into read-only / write-only.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/micro/ypattern.bin scripts/micro/ypattern.cu
#include <cstdio>
#include <cuda_runtime.h>

// B-like: read Lin rows x Q from src plane p, write Lout rows x Q to dst plane p
template <int Q>
__global__ void k_ycopy(const float2* __restrict__ src, float2* __restrict__ dst, int Nx, int Lin, int Lout,
                        int nplanes) {
    const int tiles_x = Nx / Q;
    const int ntiles = tiles_x * nplanes;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int xt = t % tiles_x, p = t / tiles_x;
        const float2* s = src + (long long)p * Lin * Nx + xt * Q;
        float2* d = dst + (long long)p * Lout * Nx + xt * Q;
        float acc = 0.f;
        for (int e = threadIdx.x; e < Lin * Q; e += blockDim.x) {
            const float2 v = __ldg(&s[(long long)(e / Q) * Nx + e % Q]);
            acc += v.x;
        }
        for (int e = threadIdx.x; e < Lout * Q; e += blockDim.x)
            d[(long long)(e / Q) * Nx + e % Q] = make_float2(acc, (float)e);
    }
}

template <int Q>
void yrun(const char* name, float2* a, float2* b, int Nx, int Lin, int Lout, int nplanes) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int occ : {4, 8}) {
        k_ycopy<Q><<<148 * occ, 256>>>(a, b, Nx, Lin, Lout, nplanes);
        cudaEventRecord(e0);
        for (int i = 0; i < 3; ++i) k_ycopy<Q><<<148 * occ, 256>>>(a, b, Nx, Lin, Lout, nplanes);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= 3;
        const double bytes = 8.0 * (Lin + Lout) * (double)Nx * nplanes;
        printf("%s Q=%2d occ=%d: %.3f ms %.0f GB/s\n", name, Q, occ, ms, bytes / ms / 1e6);
    }
}

// L2 residency: write a buffer of S bytes, then read it back in a second kernel
__global__ void k_fill(float4* p, long long n, float v) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        p[i] = make_float4(v, v, v, v);
}
__global__ void k_sum(const float4* p, long long n, float* out) {
    float a = 0.f;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        a += p[i].x;
    if (a == 12345.f) out[0] = a;
}

int main() {
    const int Nx = 2048, Ky = 1024, Ny = 2048;
    const int nplanes = 320;   // 5 comps x 64 z
    float2 *a, *b;
    cudaMalloc(&a, sizeof(float2) * (long long)nplanes * Ny * Nx);
    cudaMalloc(&b, sizeof(float2) * (long long)nplanes * Ny * Nx);
    cudaMemset(a, 0, sizeof(float2) * (long long)nplanes * Ny * Nx);
    yrun<4>("B-like (read Ky, write Ny)", a, b, Nx, Ky, Ny, nplanes);
    yrun<8>("B-like (read Ky, write Ny)", a, b, Nx, Ky, Ny, nplanes);
    yrun<16>("B-like (read Ky, write Ny)", a, b, Nx, Ky, Ny, nplanes);
    yrun<4>("D-like (read Ny, write Ky)", b, a, Nx, Ny, Ky, nplanes);
    yrun<8>("D-like (read Ny, write Ky)", b, a, Nx, Ny, Ky, nplanes);
    yrun<16>("D-like (read Ny, write Ky)", b, a, Nx, Ny, Ky, nplanes);
    // L2 residency of a freshly written buffer
    float* o;
    cudaMalloc(&o, 4);
    for (long long mb : {16LL, 32LL, 48LL, 64LL, 96LL, 2048LL}) {
        const long long n = mb * (1LL << 20) / 16;
        float4* p = reinterpret_cast<float4*>(a);
        cudaEvent_t e0, e1, e2;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventCreate(&e2);
        float ms1 = 0, ms2 = 0;
        for (int rep = 0; rep < 3; ++rep) {
            k_fill<<<148 * 8, 256>>>(reinterpret_cast<float4*>(b), (long long)1 << 28, 1.f);   // flush: 4 GB
            cudaEventRecord(e0);
            k_fill<<<148 * 8, 256>>>(p, n, 2.f);
            cudaEventRecord(e1);
            k_sum<<<148 * 8, 256>>>(p, n, o);
            cudaEventRecord(e2);
            cudaEventSynchronize(e2);
            cudaEventElapsedTime(&ms1, e0, e1);
            cudaEventElapsedTime(&ms2, e1, e2);
        }
        printf("L2 test %lld MB: write %.1f GB/s, read-after-write %.1f GB/s\n", mb, mb * 1.048576e6 / ms1 / 1e6,
               mb * 1.048576e6 / ms2 / 1e6);
    }
    return 0;
}
