// H3 (dense mode): circulant embedding + 3-D DFT of the 7 kernels,
// stored as real octant spectra.
//
// The embedding (reading G7) places T(m) at index m mod N_i for m in
// (-K_i, K_i) and zero elsewhere.  Because every kernel is even or odd along
// each axis, its N-point DFT restricted to k in [0, N/2] is a mode product
// with a real (N/2+1) x K matrix per axis:
//   even axis: C_e[k, m] = (m == 0 ? 1 : 2 cos(2 pi k m / N))
//   odd axis : C_o[k, m] = 2 sin(2 pi k m / N)          (spectrum factor -i)
// so Khat = (-i)^{#odd} T x1 C^1 x2 C^2 x3 C^3 (Eq. 11 mode products), and the
// full spectrum follows by mirror symmetry (even: Khat(N-k) = Khat(k); odd:
// Khat(N-k) = -Khat(k)).  K1c has exactly one odd axis; we store s with
// Khat1c = -i s.  Mode products run in fp64 (a tiled GEMM kernel below, setup
// only) and the result is rounded to fp32 for the hot path.

#include <cmath>
#include <vector>

#include "internal.h"

namespace svh {

namespace {
// C[b] = A[b] * op(B[b]), column-major, fp64.  A: m x k (lda), B: k x n (ldb) or,
// if TRANSB, n x k (ldb).  64x64 tiles, 256 threads, 4x4 outputs per thread.
template <bool TRANSB>
__global__ void __launch_bounds__(256) k_dgemm(int m, int n, int k, const double* __restrict__ A, int lda,
                                               long long sA, const double* __restrict__ B, int ldb, long long sB,
                                               double* __restrict__ C, int ldc, long long sC) {
    __shared__ double As[16][65];
    __shared__ double Bs[16][65];
    A += blockIdx.z * sA;
    B += blockIdx.z * sB;
    C += blockIdx.z * sC;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int m0 = blockIdx.x * 64, n0 = blockIdx.y * 64;
    double acc[4][4] = {};
    for (int k0 = 0; k0 < k; k0 += 16) {
        for (int t = threadIdx.x; t < 16 * 64; t += 256) {
            const int kk = t / 64, mm = t % 64;
            const int gm = m0 + mm, gk = k0 + kk;
            As[kk][mm] = (gm < m && gk < k) ? A[(long long)gk * lda + gm] : 0.0;
            const int gn = n0 + mm;
            double bv = 0.0;
            if (gn < n && gk < k) bv = TRANSB ? B[(long long)gk * ldb + gn] : B[(long long)gn * ldb + gk];
            Bs[kk][mm] = bv;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
            double a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk][tx + 16 * i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[kk][ty + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int gm = m0 + tx + 16 * i, gn = n0 + ty + 16 * j;
            if (gm < m && gn < n) C[(long long)gn * ldc + gm] = acc[i][j];
        }
}

void dgemm(bool transB, int m, int n, int k, const double* A, int lda, long long sA, const double* B, int ldb,
           long long sB, double* C, int ldc, long long sC, int batch) {
    dim3 grid((m + 63) / 64, (n + 63) / 64, batch);
    if (transB)
        SVH_LAUNCH(k_dgemm<true>, grid, 256, 0, 0, m, n, k, A, lda, sA, B, ldb, sB, C, ldc, sC);
    else
        SVH_LAUNCH(k_dgemm<false>, grid, 256, 0, 0, m, n, k, A, lda, sA, B, ldb, sB, C, ldc, sC);
}

std::vector<double> embed_dft_matrix(int K, int N, bool odd) {
    const int H = N / 2 + 1;
    std::vector<double> C((size_t)H * K);   // column-major H x K
    for (int m = 0; m < K; ++m)
        for (int k = 0; k < H; ++k) {
            const double th = 2.0 * M_PI * (double)((int64_t)k * m % N) / N;
            double v;
            if (odd)
                v = (m == 0) ? 0.0 : 2.0 * std::sin(th);
            else
                v = (m == 0) ? 1.0 : 2.0 * std::cos(th);
            C[(size_t)m * H + k] = v;
        }
    return C;
}

__global__ void k_to_f32(const double* __restrict__ a, float* __restrict__ b, int64_t n) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) b[i] = (float)a[i];
}
}  // namespace

// Mode products T x1 A x2 B x3 C for a tensor T[z][y][x] (x fastest) of size Kx,Ky,Kz
// with column-major matrices A (hx x Kx), B (hy x Ky), C (hz x Kz); result [hz][hy][hx].
void mode_products(const double* T, int Kx, int Ky, int Kz, const double* A, int hx, const double* B, int hy,
                   const double* C, int hz, double* w1, double* w2, double* out) {
    // mode 1: (hx x Kx) * (Kx x Ky*Kz)
    dgemm(false, hx, Ky * Kz, Kx, A, hx, 0, T, Kx, 0, w1, hx, 0, 1);
    // mode 2: per z: (hx x Ky) * (Ky x hy)
    dgemm(true, hx, hy, Ky, w1, hx, (long long)hx * Ky, B, hy, 0, w2, hx, (long long)hx * hy, Kz);
    // mode 3: (hx*hy x Kz) * (Kz x hz)
    dgemm(true, hx * hy, hz, Kz, w2, hx * hy, 0, C, hz, 0, out, hx * hy, 0, 1);
}

void compute_spectra(svh_handle* h) {
    const int K3[3] = {h->kx, h->ky, h->kz};
    const int N3[3] = {h->nx, h->ny, h->nz};
    const int H3[3] = {h->hx, h->hy, h->hz};
    double* dC[3][2];
    for (int a = 0; a < 3; ++a)
        for (int o = 0; o < 2; ++o) {
            auto C = embed_dft_matrix(K3[a], N3[a], o == 1);
            SVH_CUDA(cudaMalloc(&dC[a][o], C.size() * sizeof(double)));
            SVH_CUDA(cudaMemcpy(dC[a][o], C.data(), C.size() * sizeof(double), cudaMemcpyHostToDevice));
        }
    const int64_t n1 = (int64_t)h->hx * h->ky * h->kz, n2 = (int64_t)h->hx * h->hy * h->kz;
    const int64_t no = (int64_t)h->hx * h->hy * h->hz;
    double *w1, *w2, *wo;
    SVH_CUDA(cudaMalloc(&w1, n1 * sizeof(double)));
    SVH_CUDA(cudaMalloc(&w2, n2 * sizeof(double)));
    SVH_CUDA(cudaMalloc(&wo, no * sizeof(double)));
    SVH_CUDA(cudaMalloc(&h->d_spec, 7 * no * sizeof(float)));
    if (h->opts.precision == 1) SVH_CUDA(cudaMalloc(&h->d_spec64, 7 * no * sizeof(double)));   // complex128 build
    // kernel order K0, K1x, K1y, K1z, K2x, K2y, K2z; odd axis of K1c is c
    for (int q = 0; q < 7; ++q) {
        const int odd_axis = (q >= 1 && q <= 3) ? q - 1 : -1;
        mode_products(h->d_kern + q * h->Kt, h->kx, h->ky, h->kz, dC[0][odd_axis == 0], H3[0],
                      dC[1][odd_axis == 1], H3[1], dC[2][odd_axis == 2], H3[2], w1, w2, wo);
        SVH_LAUNCH(k_to_f32, dim3((unsigned)((no + 255) / 256)), 256, 0, 0, wo, h->d_spec + q * no, no);
        if (h->d_spec64) SVH_CUDA(cudaMemcpy(h->d_spec64 + q * no, wo, no * sizeof(double), cudaMemcpyDeviceToDevice));
    }
    SVH_CUDA(cudaDeviceSynchronize());
    cudaFree(w1);
    cudaFree(w2);
    cudaFree(wo);
    for (int a = 0; a < 3; ++a)
        for (int o = 0; o < 2; ++o) cudaFree(dC[a][o]);
}

void dgemm_nt(int m, int n, int k, const double* A, int lda, const double* B, int ldb, double* C, int ldc) {
    dgemm(true, m, n, k, A, lda, 0, B, ldb, 0, C, ldc, 0, 1);
}
std::vector<double> embed_dft_matrix_host(int K, int N, bool odd) { return embed_dft_matrix(K, N, odd); }

}  // namespace svh
