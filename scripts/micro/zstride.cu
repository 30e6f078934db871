// Micro-benchmark: pass C's tile pattern (Q consecutive kx x Kz "planes" x 5 components,
// read-modify-write) as a function of the distance between consecutive z rows of a tile.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/micro/zstride.bin scripts/micro/zstride.cu
#include <cstdio>
#include <cuda_runtime.h>

// element (rc, z, ky, kx) at rc*RC + blk(ky)*BS + z*ZS + in(ky)*Nx + kx with ky = blk*B + in
template <int Q>
__global__ void k_rmw(float2* X, int Nx, int Ny, int Kz, int B, long long ZS, long long BS, long long RC, int ntiles) {
    const int tiles_x = Nx / Q;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int xt = t % tiles_x, rest = t / tiles_x;
        const int ky = rest % Ny, r = rest / Ny;
        float2* base = X + (long long)r * 5 * RC + (long long)(ky / B) * BS + (long long)(ky % B) * Nx + xt * Q;
        for (int e = threadIdx.x; e < 5 * Kz * Q; e += blockDim.x) {
            const int q = e % Q, row = e / Q, z = row % Kz, c = row / Kz;
            float2* p = base + (long long)c * RC + (long long)z * ZS + q;
            float2 v = *p;
            v.x = v.x * 1.0001f + 1.f;
            *p = v;
        }
    }
}

template <int Q>
void run(float2* X, int Nx, int Ny, int Kz, int B) {
    const long long ZS = (long long)B * Nx, BS = (long long)Kz * B * Nx, RC = (long long)Kz * Ny * Nx;
    const int ntiles = (Nx / Q) * Ny * 2;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_rmw<Q><<<148 * 8, 256>>>(X, Nx, Ny, Kz, B, ZS, BS, RC, ntiles);
    cudaEventRecord(a);
    for (int i = 0; i < 3; ++i) k_rmw<Q><<<148 * 8, 256>>>(X, Nx, Ny, Kz, B, ZS, BS, RC, ntiles);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ms /= 3;
    const double bytes = 2.0 * 8 * 5 * Kz * (double)Nx * Ny * 2;
    printf("Q=%2d ky-block B=%4d (z stride %8lld B): %.3f ms %.0f GB/s\n", Q, B, ZS * 8, ms, bytes / ms / 1e6);
}

int main() {
    const int Nx = 2048, Ny = 2048, Kz = 64;
    float2* X;
    const size_t n = (size_t)2 * 5 * Kz * Ny * Nx;
    cudaMalloc(&X, n * sizeof(float2));
    cudaMemset(X, 0, n * sizeof(float2));
    for (int B : {1, 8, 64, 256, 2048}) {
        run<8>(X, Nx, Ny, Kz, B);
        run<16>(X, Nx, Ny, Kz, B);
        run<32>(X, Nx, Ny, Kz, B);
    }
    return 0;
}
