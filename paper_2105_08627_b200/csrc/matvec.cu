// FFT-circulant VIE matvec, Eq. 9:
//   CC^b = z^b I^b + IFFT{ sum_a Zhat^{b,a} * FFT(I^a) }   (cropped to the voxels)
//
// Plan P5: five passes over HBM per right-hand side,
//   A  x: scatter/zero-pad (gather from packed order) + forward FFT along x   Kt -> 2Kt pts/comp
//   B  y: zero-pad + forward FFT along y (strided pencils)                    2Kt -> 4Kt
//   C  z: zero-pad + forward FFT along z, 5->5 moment-form MAC with the 7
//         kernel spectra (dense octant or Tucker-expanded), inverse FFT, crop  4Kt -> 4Kt (in place)
//   D  y: inverse FFT along y + crop                                          4Kt -> 2Kt
//   E  x: inverse FFT along x + crop + local term z^b I^b + scatter to packed 2Kt -> Kt
// The circulant spectra never exist densely in HBM in Tucker mode; in dense
// mode only the 7 real octant spectra (Kt-sized, fp32) are read.
#include <algorithm>
#include <cuda_runtime.h>

#include "fft.cuh"
#include "internal.h"

namespace svh {

// ---------------------------------------------------------------------------
// Pass A: rows along x (contiguous).  S[j*PP + q], q = row within the tile.
template <int N, bool PACKED>
__global__ void __launch_bounds__(fft_max_threads(N)) k_pass_a(const float2* __restrict__ in, float2* __restrict__ X1,
                                                const int32_t* __restrict__ vmap, const float2* __restrict__ tw,
                                                int Kx, int rows, int64_t K, int64_t Kt, int Q) {
    extern __shared__ float2 S[];
    const int PP = Q + 1;
    const int rc = blockIdx.y;
    const int row0 = blockIdx.x * Q;
    const int nq = min(Q, rows - row0);
    for (int t = threadIdx.x; t < Q * N; t += blockDim.x) {
        const int q = t / N, j = t - (t / N) * N;
        float2 v = make_float2(0.f, 0.f);
        if (q < nq && j < Kx) {
            const int64_t cell = (int64_t)(row0 + q) * Kx + j;
            const int idx = __ldg(&vmap[cell]);
            if (idx >= 0) v = PACKED ? in[(int64_t)rc * K + idx] : in[(int64_t)rc * Kt + cell];
        }
        S[j * PP + q] = v;
    }
    __syncthreads();
    smem_fft<N, -1>(S, PP, Q, tw);
    for (int t = threadIdx.x; t < Q * N; t += blockDim.x) {
        const int q = t / N, j = t - (t / N) * N;
        if (q < nq) X1[((int64_t)rc * rows + row0 + q) * N + j] = S[j * PP + q];
    }
}

// Pass B / D: pencils along y (stride Nx).  Tile = Q consecutive kx at one (z, rc).
template <int N, int DIR>
__global__ void __launch_bounds__(fft_max_threads(N)) k_pass_y(const float2* __restrict__ in, float2* __restrict__ out,
                                                const float2* __restrict__ tw, int Nx, int Kz, int Lin,
                                                int Lout, int Q) {
    extern __shared__ float2 S[];
    const int PP = Q + 1;
    const int kx0 = blockIdx.x * Q;
    const int z = blockIdx.y;
    const int64_t rc = blockIdx.z;
    const float2* src = in + ((rc * Kz + z) * Lin) * (int64_t)Nx + kx0;
    float2* dst = out + ((rc * Kz + z) * Lout) * (int64_t)Nx + kx0;
    const int nq = min(Q, Nx - kx0);
    for (int t = threadIdx.x; t < Q * N; t += blockDim.x) {
        const int j = t / Q, q = t - (t / Q) * Q;
        float2 v = make_float2(0.f, 0.f);
        if (j < Lin && q < nq) v = src[(int64_t)j * Nx + q];
        S[j * PP + q] = v;
    }
    __syncthreads();
    smem_fft<N, DIR>(S, PP, Q, tw);
    for (int t = threadIdx.x; t < Q * Lout; t += blockDim.x) {
        const int j = t / Q, q = t - (t / Q) * Q;
        if (q < nq) dst[(int64_t)j * Nx + q] = S[j * PP + q];
    }
}

// Moment-form 5->5 multiply-accumulate at one frequency point:
//   m1x = I2D + I3D, m1y = I3D - I2D, m1z = -2 I3D
//   P0c = K0 Ic + K1c m1c,  P1c = -K1c Ic + K2c m1c     (c = x, y, z)
//   CC^c = P0c, CC^2D = P1x - P1y, CC^3D = P1x + P1y - 2 P1z
// with Khat0, Khat2 real and Khat1c = -i s1c (odd kernels have imaginary spectra).
// The whole Green sum is multiplied by j * omega mu0 dx / (Nx Ny Nz).
__device__ __forceinline__ void mac5(float2 (&v)[5], float k0, float s1x, float s1y, float s1z, float k2x,
                                     float k2y, float k2z, float g) {
    const float2 Ix = v[0], Iy = v[1], Iz = v[2], I2 = v[3], I3 = v[4];
    const float2 m1x = cadd(I2, I3), m1y = csub(I3, I2), m1z = cscale(I3, -2.f);
    // K1 m = -i s m ;  -K1 I = +i s I
    const float2 P0x = cadd(cscale(Ix, k0), cmul_i(m1x, -s1x));
    const float2 P0y = cadd(cscale(Iy, k0), cmul_i(m1y, -s1y));
    const float2 P0z = cadd(cscale(Iz, k0), cmul_i(m1z, -s1z));
    const float2 P1x = cadd(cmul_i(Ix, s1x), cscale(m1x, k2x));
    const float2 P1y = cadd(cmul_i(Iy, s1y), cscale(m1y, k2y));
    const float2 P1z = cadd(cmul_i(Iz, s1z), cscale(m1z, k2z));
    const float2 C2 = csub(P1x, P1y);
    const float2 C3 = csub(cadd(P1x, P1y), cscale(P1z, 2.f));
    // multiply by j*g
    v[0] = cmul_i(P0x, g);
    v[1] = cmul_i(P0y, g);
    v[2] = cmul_i(P0z, g);
    v[3] = cmul_i(C2, g);
    v[4] = cmul_i(C3, g);
}

struct SpecView {
    const float* spec;   // dense [7][hz][hy][hx]
    int hx, hy, hz;
};

// Pass C: pencils along z (stride Nx*Ny), all 5 components of Q consecutive kx at one ky.
template <int N>
__global__ void __launch_bounds__(fft_max_threads(N)) k_pass_c(float2* __restrict__ X2, SpecView sv,
                                                const float2* __restrict__ tw, int Nx, int Ny, int Kz, int Q,
                                                float g) {
    extern __shared__ float2 S[];
    const int Q5 = 5 * Q;
    const int PP = Q5 + 1;
    const int kx0 = blockIdx.x * Q;
    const int ky = blockIdx.y;
    const int64_t r = blockIdx.z;
    const int64_t plane = (int64_t)Nx * Ny;
    float2* base = X2 + r * 5 * Kz * plane + (int64_t)ky * Nx + kx0;
    const int nq = min(Q, Nx - kx0);
    for (int t = threadIdx.x; t < Q * N * 5; t += blockDim.x) {
        const int q = t % Q;
        const int rest = t / Q;
        const int j = rest % N, c = rest / N;
        float2 v = make_float2(0.f, 0.f);
        if (j < Kz && q < nq) v = base[((int64_t)c * Kz + j) * plane + q];
        S[j * PP + c * Q + q] = v;
    }
    __syncthreads();
    smem_fft<N, -1>(S, PP, Q5, tw);
    // frequency-domain block multiply-accumulate
    const int nxh = Nx >> 1, nyh = Ny >> 1, nzh = N >> 1;
    const int oy = ky <= nyh ? ky : Ny - ky;
    const float sy = ky <= nyh ? 1.f : -1.f;
    for (int t = threadIdx.x; t < Q * N; t += blockDim.x) {
        const int q = t % Q, kz = t / Q;
        const int kx = kx0 + q;
        if (q >= nq) continue;
        const int ox = kx <= nxh ? kx : Nx - kx;
        const float sx = kx <= nxh ? 1.f : -1.f;
        const int oz = kz <= nzh ? kz : N - kz;
        const float sz = kz <= nzh ? 1.f : -1.f;
        float kv[7];
        const int64_t pl = (int64_t)sv.hx * sv.hy * sv.hz;
        const int64_t o = ((int64_t)oz * sv.hy + oy) * sv.hx + ox;
#pragma unroll
        for (int k = 0; k < 7; ++k) kv[k] = __ldg(&sv.spec[k * pl + o]);
        float2 v[5];
#pragma unroll
        for (int c = 0; c < 5; ++c) v[c] = S[kz * PP + c * Q + q];
        mac5(v, kv[0], sx * kv[1], sy * kv[2], sz * kv[3], kv[4], kv[5], kv[6], g);
#pragma unroll
        for (int c = 0; c < 5; ++c) S[kz * PP + c * Q + q] = v[c];
    }
    __syncthreads();
    smem_fft<N, +1>(S, PP, Q5, tw);
    for (int t = threadIdx.x; t < Q * Kz * 5; t += blockDim.x) {
        const int q = t % Q;
        const int rest = t / Q;
        const int j = rest % Kz, c = rest / Kz;
        if (q < nq) base[((int64_t)c * Kz + j) * plane + q] = S[j * PP + c * Q + q];
    }
}

// Pass E: rows along x, inverse FFT, crop, local term, scatter.
template <int N, bool PACKED>
__global__ void __launch_bounds__(fft_max_threads(N)) k_pass_e(const float2* __restrict__ X1, float2* __restrict__ out,
                                                const float2* __restrict__ in, const int32_t* __restrict__ vmap,
                                                const uint8_t* __restrict__ mat, const float2* __restrict__ zloc,
                                                const float2* __restrict__ tw, int Kx, int rows, int64_t K,
                                                int64_t Kt, int Q, int green_only) {
    extern __shared__ float2 S[];
    const int PP = Q + 1;
    const int rc = blockIdx.y;
    const int comp = rc % 5;
    const int row0 = blockIdx.x * Q;
    const int nq = min(Q, rows - row0);
    for (int t = threadIdx.x; t < Q * N; t += blockDim.x) {
        const int q = t / N, j = t - (t / N) * N;
        float2 v = make_float2(0.f, 0.f);
        if (q < nq) v = X1[((int64_t)rc * rows + row0 + q) * N + j];
        S[j * PP + q] = v;
    }
    __syncthreads();
    smem_fft<N, +1>(S, PP, Q, tw);
    for (int t = threadIdx.x; t < Q * Kx; t += blockDim.x) {
        const int q = t / Kx, j = t - (t / Kx) * Kx;
        if (q >= nq) continue;
        const int64_t cell = (int64_t)(row0 + q) * Kx + j;
        const int idx = __ldg(&vmap[cell]);
        if (idx < 0) {
            if (!PACKED) out[(int64_t)rc * Kt + cell] = make_float2(0.f, 0.f);
            continue;
        }
        float2 v = S[j * PP + q];
        if (!green_only) {
            const float2 z = __ldg(&zloc[mat[cell] * 5 + comp]);
            const float2 iv = PACKED ? in[(int64_t)rc * K + idx] : in[(int64_t)rc * Kt + cell];
            v = cadd(v, cmul(z, iv));
        }
        if (PACKED)
            out[(int64_t)rc * K + idx] = v;
        else
            out[(int64_t)rc * Kt + cell] = v;
    }
}

// ---------------------------------------------------------------------------
// host-side dispatch
namespace {

template <typename F>
void set_smem(F* kern, size_t bytes) {
    if (bytes > 48 * 1024) SVH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

constexpr size_t kSmemCap = 110 * 1024;

int pick_q(int N, int want_threads, int multiplicity, int qmax) {
    const int tpp = fft_threads_per_pencil(N);
    want_threads = std::min(want_threads, fft_max_threads(N));
    int Q = std::max(1, want_threads / (tpp * multiplicity));
    while (Q > 1 && (size_t)N * (multiplicity * Q + 1) * sizeof(float2) > kSmemCap) Q >>= 1;
    return std::max(1, std::min(Q, qmax));
}

template <int N>
void run_pass_a(svh_handle* h, const float2* in, bool packed, int nrhs, cudaStream_t s) {
    const int rows = h->ky * h->kz;
    const int Q = pick_q(N, 256, 1, rows);
    const int nt = std::max(32, fft_threads_per_pencil(N) * Q);
    const size_t smem = (size_t)N * (Q + 1) * sizeof(float2);
    dim3 grid((rows + Q - 1) / Q, 5 * nrhs);
    if (packed) {
        set_smem((k_pass_a<N, true>), smem);
        SVH_LAUNCH((k_pass_a<N, true>), grid, nt, smem, s, in, h->X1, h->d_vmap, h->d_tw[0], h->kx, rows, h->K, h->Kt, Q);
    } else {
        set_smem((k_pass_a<N, false>), smem);
        SVH_LAUNCH((k_pass_a<N, false>), grid, nt, smem, s, in, h->X1, h->d_vmap, h->d_tw[0], h->kx, rows, h->K, h->Kt, Q);
    }
}

template <int N, int DIR>
void run_pass_y(svh_handle* h, const float2* in, float2* out, int Lin, int Lout, int nrhs, cudaStream_t s) {
    const int Q = pick_q(N, 256, 1, std::max(1, h->nx));
    const int nt = std::max(32, fft_threads_per_pencil(N) * Q);
    const size_t smem = (size_t)N * (Q + 1) * sizeof(float2);
    dim3 grid((h->nx + Q - 1) / Q, h->kz, 5 * nrhs);
    set_smem((k_pass_y<N, DIR>), smem);
    SVH_LAUNCH((k_pass_y<N, DIR>), grid, nt, smem, s, in, out, h->d_tw[1], h->nx, h->kz, Lin, Lout, Q);
}

template <int N>
void run_pass_c(svh_handle* h, int nrhs, cudaStream_t s) {
    const int Q = pick_q(N, 320, 5, std::max(1, h->nx));
    const int nt = std::max(32, fft_threads_per_pencil(N) * 5 * Q);
    const size_t smem = (size_t)N * (5 * Q + 1) * sizeof(float2);
    dim3 grid((h->nx + Q - 1) / Q, h->ny, nrhs);
    SpecView sv{};
    sv.spec = h->d_spec;
    sv.hx = h->hx;
    sv.hy = h->hy;
    sv.hz = h->hz;
    set_smem(k_pass_c<N>, smem);
    SVH_LAUNCH((k_pass_c<N>), grid, nt, smem, s, h->X2, sv, h->d_tw[2], h->nx, h->ny, h->kz, Q, h->gscale);
}

template <int N>
void run_pass_e(svh_handle* h, const float2* in, float2* out, bool packed, bool green_only, int nrhs,
                cudaStream_t s) {
    const int rows = h->ky * h->kz;
    const int Q = pick_q(N, 256, 1, rows);
    const int nt = std::max(32, fft_threads_per_pencil(N) * Q);
    const size_t smem = (size_t)N * (Q + 1) * sizeof(float2);
    dim3 grid((rows + Q - 1) / Q, 5 * nrhs);
    if (packed) {
        set_smem((k_pass_e<N, true>), smem);
        SVH_LAUNCH((k_pass_e<N, true>), grid, nt, smem, s, h->X1, out, in, h->d_vmap, h->d_mat, h->d_zloc, h->d_tw[0],
                   h->kx, rows, h->K, h->Kt, Q, (int)green_only);
    } else {
        set_smem((k_pass_e<N, false>), smem);
        SVH_LAUNCH((k_pass_e<N, false>), grid, nt, smem, s, h->X1, out, in, h->d_vmap, h->d_mat, h->d_zloc, h->d_tw[0],
                   h->kx, rows, h->K, h->Kt, Q, (int)green_only);
    }
}

#define SVH_DISPATCH_N(n, CALL)                   \
    switch (n) {                                  \
        case 1: { constexpr int NN = 1; CALL; break; }       \
        case 2: { constexpr int NN = 2; CALL; break; }       \
        case 4: { constexpr int NN = 4; CALL; break; }       \
        case 8: { constexpr int NN = 8; CALL; break; }       \
        case 16: { constexpr int NN = 16; CALL; break; }     \
        case 32: { constexpr int NN = 32; CALL; break; }     \
        case 64: { constexpr int NN = 64; CALL; break; }     \
        case 128: { constexpr int NN = 128; CALL; break; }   \
        case 256: { constexpr int NN = 256; CALL; break; }   \
        case 512: { constexpr int NN = 512; CALL; break; }   \
        case 1024: { constexpr int NN = 1024; CALL; break; } \
        case 2048: { constexpr int NN = 2048; CALL; break; } \
        case 4096: { constexpr int NN = 4096; CALL; break; } \
        default: throw Error{SVH_EINVAL, "embedding extent not supported (max 4096)"}; \
    }

}  // namespace

void ensure_workspace(svh_handle* h, int nrhs) {
    if (h->ws_rhs >= nrhs) return;
    if (h->X1) cudaFree(h->X1);
    if (h->X2) cudaFree(h->X2);
    h->X1 = h->X2 = nullptr;
    h->ws_rhs = 0;
    const size_t n1 = (size_t)nrhs * 5 * h->kz * h->ky * h->nx;
    const size_t n2 = (size_t)nrhs * 5 * h->kz * h->ny * h->nx;
    if (cudaMalloc(&h->X1, n1 * sizeof(float2)) != cudaSuccess ||
        cudaMalloc(&h->X2, n2 * sizeof(float2)) != cudaSuccess) {
        cudaGetLastError();
        if (h->X1) cudaFree(h->X1);
        h->X1 = nullptr;
        throw Error{SVH_ENOMEM, "matvec workspace allocation failed"};
    }
    h->ws_rhs = nrhs;
}

int max_chunk(svh_handle* h) {
    if (h->opts.rhs_chunk > 0) return h->opts.rhs_chunk;
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    const size_t per = (size_t)5 * h->kz * (h->ky + h->ny) * h->nx * sizeof(float2);
    size_t budget = (size_t)(0.5 * (double)(fr + (size_t)h->ws_rhs * per));
    return (int)std::max<size_t>(1, std::min<size_t>(64, budget / per));
}

void matvec(svh_handle* h, const float2* I, float2* CC, int nrhs, bool green_only, bool packed, cudaStream_t s) {
    const int chunk = std::min(nrhs, max_chunk(h));
    ensure_workspace(h, chunk);
    const int64_t per_rhs = 5 * (packed ? h->K : h->Kt);
    for (int r0 = 0; r0 < nrhs; r0 += chunk) {
        const int nr = std::min(chunk, nrhs - r0);
        const float2* in = I + r0 * per_rhs;
        float2* out = CC + r0 * per_rhs;
        SVH_DISPATCH_N(h->nx, run_pass_a<NN>(h, in, packed, nr, s));
        SVH_DISPATCH_N(h->ny, (run_pass_y<NN, -1>(h, h->X1, h->X2, h->ky, h->ny, nr, s)));
        SVH_DISPATCH_N(h->nz, run_pass_c<NN>(h, nr, s));
        SVH_DISPATCH_N(h->ny, (run_pass_y<NN, +1>(h, h->X2, h->X1, h->ny, h->ky, nr, s)));
        SVH_DISPATCH_N(h->nx, run_pass_e<NN>(h, in, out, packed, green_only, nr, s));
    }
}

}  // namespace svh
