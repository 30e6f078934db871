// Micro-benchmark: achievable HBM bandwidth of pass C's access pattern (read-modify-write of
// tiles of Q consecutive kx x Kz planes x 5 components, plane stride S) -- pure data movement.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/zpattern scripts/micro/zpattern.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int Q>
__global__ void k_tile_rmw(float2* X, long long plane, int Nx, int Ny, int Kz, int ntiles) {
    // one warp-group per tile: thread (z-lane, q); each tile: 5*Kz rows of Q elements
    const int tiles_x = Nx / Q;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int xt = t % tiles_x, rest = t / tiles_x;
        const int ky = rest % Ny, r = rest / Ny;
        float2* base = X + (long long)r * 5 * Kz * plane + (long long)ky * Nx + xt * Q;
        for (int e = threadIdx.x; e < 5 * Kz * Q; e += blockDim.x) {
            const int q = e % Q, row = e / Q;
            float2* p = base + (long long)row * plane + q;
            float2 v = *p;
            v.x = v.x * 1.0001f + 1.f;
            *p = v;
        }
    }
}

template <int Q>
void run(float2* X, long long plane, int Nx, int Ny, int Kz, int R) {
    const int ntiles = (Nx / Q) * Ny * R;
    int nt = 256;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int occ : {2, 4, 8}) {
        k_tile_rmw<Q><<<148 * occ, nt>>>(X, plane, Nx, Ny, Kz, ntiles);
        cudaEventRecord(a);
        for (int i = 0; i < 3; ++i) k_tile_rmw<Q><<<148 * occ, nt>>>(X, plane, Nx, Ny, Kz, ntiles);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        ms /= 3;
        const double bytes = 2.0 * 8 * 5 * Kz * (double)Nx * Ny * R;
        printf("Q=%2d plane=%lld occ=%d: %.3f ms  %.0f GB/s\n", Q, plane, occ, ms, bytes / ms / 1e6);
    }
}

int main() {
    const int Nx = 2048, Ny = 2048, Kz = 64, R = 2;
    for (long long pad : {0LL, 64LL, 1000LL}) {
        const long long plane = (long long)Nx * Ny + pad;
        float2* X;
        cudaMalloc(&X, sizeof(float2) * plane * 5 * Kz * R + 4096);
        cudaMemset(X, 0, sizeof(float2) * plane * 5 * Kz * R);
        run<4>(X, plane, Nx, Ny, Kz, R);
        run<8>(X, plane, Nx, Ny, Kz, R);
        run<16>(X, plane, Nx, Ny, Kz, R);
        run<32>(X, plane, Nx, Ny, Kz, R);
        cudaFree(X);
    }
    return 0;
}
