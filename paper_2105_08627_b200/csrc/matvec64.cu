// The complex128 build of the matvec (svh_opts.precision = 1; SURVEY 8(b) "precision c64|c128",
// 8(c) c.5 "GPU fp64 build <= 1e-12"): Eq. 9 in double precision with the dense fp64
// octant spectra, for tight solves (the paper runs MATLAB double) and as the fp64
// reference the c64 product is compared with on the GPU.
//
// Deliberately plain: scatter into the full embedding W = [rc][Nz][Ny][Nx], radix-2 FFTs of
// pencils staged in shared memory along x, y, z (TI pencils per CTA, coalesced along the
// contiguous index), the 5 -> 5 moment-form MAC per frequency point (7 fp64 kernel values from
// the octant by mirror symmetry), inverse FFTs z, y, x, gather + local term.  It is a
// correctness path (fp64 tensor cores are not on B200's roofline, and the c64 passes are the
// product), so it carries no pruning.
#include <algorithm>
#include <cuda_runtime.h>

#include "internal.h"

namespace svh {
namespace {

constexpr int kF64Threads = 256;
constexpr int kF64Smem = 64 * 1024;   // bytes of pencil staging per CTA

__device__ __forceinline__ double2 zmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// embedding cell of the lattice cell c (x fastest over Kx, Ky, Kz)
__device__ __forceinline__ int64_t emb_cell(int64_t c, int Kx, int Ky, int Nx, int Ny) {
    const int64_t x = c % Kx, r = c / Kx;
    const int64_t y = r % Ky, z = r / Ky;
    return (z * Ny + y) * Nx + x;
}

__global__ void k64_scatter_emb(const double2* __restrict__ I, double2* __restrict__ W,
                                const int32_t* __restrict__ vox, int64_t K, int64_t Nt, int nrc, int Kx, int Ky,
                                int Nx, int Ny) {
    const int64_t n = (int64_t)nrc * K;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t rc = e / K, k = e - rc * K;
        W[rc * Nt + emb_cell(__ldg(&vox[k]), Kx, Ky, Nx, Ny)] = I[e];
    }
}

// In-place FFTs of length N (power of two) of the pencils (o, i): element j at
// o so + i si + j sj, i < ni; TI pencils of one o per CTA, staged bit-reversed in shared memory,
// radix-2 DIT stages; tw[j] = exp(-2 pi i j / N) (fp64); DIR = -1 forward, +1 inverse (unscaled).
template <int DIR>
__global__ void __launch_bounds__(kF64Threads)
    k64_fft(double2* __restrict__ W, int N, int lg, int64_t so, int64_t si, int64_t sj, int64_t no, int64_t ni,
            int TI, const double2* __restrict__ tw) {
    extern __shared__ double2 S[];   // [TI][N]
    const int64_t nib = (ni + TI - 1) / TI;
    for (int64_t g = blockIdx.x; g < no * nib; g += gridDim.x) {
        const int64_t o = g / nib, i0 = (g % nib) * TI;
        const int tn = (int)std::min<int64_t>(TI, ni - i0);
        __syncthreads();
        for (int e = threadIdx.x; e < TI * N; e += blockDim.x) {
            int t, j;
            if (si == 1) {   // consecutive threads -> consecutive i (contiguous)
                t = e % TI;
                j = e / TI;
            } else {         // consecutive threads -> consecutive j
                t = e / N;
                j = e % N;
            }
            if (t < tn) S[t * N + (int)(__brev((unsigned)j) >> (32 - lg))] = W[o * so + (i0 + t) * si + (int64_t)j * sj];
        }
        __syncthreads();
        for (int len = 2; len <= N; len <<= 1) {
            const int half = len >> 1, step = N / len;
            for (int b = threadIdx.x; b < tn * (N / 2); b += blockDim.x) {
                const int t = b / (N / 2), r = b % (N / 2);
                const int k = r % half, i1 = (r / half) * len + k;
                double2 w = __ldg(&tw[k * step]);
                if (DIR > 0) w.y = -w.y;
                const double2 u = S[t * N + i1], v = zmul(S[t * N + i1 + half], w);
                S[t * N + i1] = make_double2(u.x + v.x, u.y + v.y);
                S[t * N + i1 + half] = make_double2(u.x - v.x, u.y - v.y);
            }
            __syncthreads();
        }
        for (int e = threadIdx.x; e < TI * N; e += blockDim.x) {
            int t, j;
            if (si == 1) {
                t = e % TI;
                j = e / TI;
            } else {
                t = e / N;
                j = e % N;
            }
            if (t < tn) W[o * so + (i0 + t) * si + (int64_t)j * sj] = S[t * N + j];
        }
    }
}

// 5 -> 5 moment-form MAC at every frequency point of the embedding, fp64
__global__ void k64_mac(double2* __restrict__ W, int nrhs, int Nx, int Ny, int Nz, const double* __restrict__ spec,
                        int hx, int hy, int hz, double g) {
    const int64_t Nt = (int64_t)Nx * Ny * Nz;
    const int64_t pl = (int64_t)hx * hy * hz;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)nrhs * Nt;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e / Nt, p = e - r * Nt;
        const int kx = (int)(p % Nx), ky = (int)((p / Nx) % Ny), kz = (int)(p / ((int64_t)Nx * Ny));
        const int ox = kx <= Nx / 2 ? kx : Nx - kx, oy = ky <= Ny / 2 ? ky : Ny - ky, oz = kz <= Nz / 2 ? kz : Nz - kz;
        const double sx = kx <= Nx / 2 ? 1.0 : -1.0, sy = ky <= Ny / 2 ? 1.0 : -1.0, sz = kz <= Nz / 2 ? 1.0 : -1.0;
        const int64_t o = ((int64_t)oz * hy + oy) * hx + ox;
        const double f0 = g * spec[0 * pl + o], f1 = g * sx * spec[1 * pl + o], f2 = g * sy * spec[2 * pl + o];
        const double f3 = -2.0 * g * sz * spec[3 * pl + o];
        const double f4 = g * spec[4 * pl + o], f5 = g * spec[5 * pl + o], f6 = 4.0 * g * spec[6 * pl + o];
        double2* w = W + r * 5 * Nt + p;
        const double2 Ix = w[0], Iy = w[Nt], Iz = w[2 * Nt], I2 = w[3 * Nt], I3 = w[4 * Nt];
        const double2 m1x = make_double2(I2.x + I3.x, I2.y + I3.y), m1y = make_double2(I3.x - I2.x, I3.y - I2.y);
        auto ims = [](double2 a, double s) { return make_double2(-a.y * s, a.x * s); };   // a * (i s)
        auto axs = [](double2 a, double s, double2 b) { return make_double2(b.x + a.x * s, b.y + a.y * s); };
        const double2 Qx = axs(Ix, -f1, ims(m1x, f4));
        const double2 Qy = axs(Iy, -f2, ims(m1y, f5));
        const double2 Qz = axs(Iz, -f3, ims(I3, f6));
        w[0] = axs(m1x, f1, ims(Ix, f0));
        w[Nt] = axs(m1y, f2, ims(Iy, f0));
        w[2 * Nt] = axs(I3, f3, ims(Iz, f0));
        w[3 * Nt] = make_double2(Qx.x - Qy.x, Qx.y - Qy.y);
        w[4 * Nt] = make_double2(Qx.x + Qy.x + Qz.x, Qx.y + Qy.y + Qz.y);
    }
}

__global__ void k64_gather(const double2* __restrict__ W, const double2* __restrict__ I, double2* __restrict__ out,
                           const int32_t* __restrict__ vox, const uint8_t* __restrict__ matp,
                           const double2* __restrict__ zloc, int64_t K, int64_t Nt, int nrc, int Kx, int Ky, int Nx,
                           int Ny, int green_only) {
    const int64_t n = (int64_t)nrc * K;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t rc = e / K, k = e - rc * K;
        const int c = (int)(rc % 5);
        double2 v = W[rc * Nt + emb_cell(__ldg(&vox[k]), Kx, Ky, Nx, Ny)];
        if (!green_only) {
            const double2 z = zloc[(int)__ldg(&matp[k]) * 5 + c];
            const double2 zi = zmul(z, I[e]);
            v = make_double2(v.x + zi.x, v.y + zi.y);
        }
        out[e] = v;
    }
}

int blocks_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)); }

void fft_axis(svh_handle* h, double2* W, int nrhs, int axis, int dir, cudaStream_t s) {
    const int N3[3] = {h->nx, h->ny, h->nz};
    const int N = N3[axis];
    if (N == 1) return;
    const int64_t Nx = h->nx, Ny = h->ny, Nz = h->nz, Nt = Nx * Ny * Nz;
    int64_t so, si, sj, no, ni;
    if (axis == 0) {
        so = 0, si = Nx, sj = 1, no = 1, ni = (int64_t)5 * nrhs * Nz * Ny;
    } else if (axis == 1) {
        so = Ny * Nx, si = 1, sj = Nx, no = (int64_t)5 * nrhs * Nz, ni = Nx;
    } else {
        so = Nt, si = 1, sj = Ny * Nx, no = (int64_t)5 * nrhs, ni = Ny * Nx;
    }
    const int TI = std::max(1, std::min(64, kF64Smem / (int)(N * sizeof(double2))));
    const size_t smem = (size_t)TI * N * sizeof(double2);
    const int lg = ilog2(N);
    const int64_t groups = no * ((ni + TI - 1) / TI);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(groups, 148 * 8));
    auto go = [&](auto kern) {
        SVH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        SVH_LAUNCH(kern, grid, kF64Threads, smem, s, W, N, lg, so, si, sj, no, ni, TI, h->d_tw64[axis]);
    };
    if (dir < 0)
        go(k64_fft<-1>);
    else
        go(k64_fft<+1>);
}

}  // namespace

void matvec_z(svh_handle* h, const double2* I, double2* CC, int nrhs, bool green_only, cudaStream_t s) {
    SVH_CHECK(h->opts.precision == 1 && h->d_spec64, SVH_EINVAL,
              "the complex128 matvec needs a handle set up with opts.precision = 1");
    const int64_t Nt = (int64_t)h->nx * h->ny * h->nz;
    const size_t per = (size_t)5 * Nt * sizeof(double2);
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    const int cap = (int)std::max<size_t>(1, std::min<size_t>((size_t)nrhs, (size_t)(0.6 * (double)(fr + h->w64_bytes)) / per));
    if (h->w64_bytes < (size_t)cap * per) {
        cudaFree(h->W64);
        h->W64 = nullptr;
        h->w64_bytes = 0;
        SVH_CUDA(cudaMalloc(&h->W64, (size_t)cap * per));
        h->w64_bytes = (size_t)cap * per;
    }
    double2* W = h->W64;
    for (int r0 = 0; r0 < nrhs; r0 += cap) {
        const int nr = std::min(cap, nrhs - r0);
        const double2* in = I + (int64_t)r0 * 5 * h->K;
        double2* out = CC + (int64_t)r0 * 5 * h->K;
        SVH_CUDA(cudaMemsetAsync(W, 0, (size_t)nr * per, s));
        SVH_LAUNCH(k64_scatter_emb, blocks_for((int64_t)5 * nr * h->K), 256, 0, s, in, W, h->d_vox, h->K, Nt, 5 * nr,
                   h->kx, h->ky, h->nx, h->ny);
        for (int a = 0; a < 3; ++a) fft_axis(h, W, nr, a, -1, s);
        SVH_LAUNCH(k64_mac, blocks_for((int64_t)nr * Nt), 256, 0, s, W, nr, h->nx, h->ny, h->nz, h->d_spec64, h->hx,
                   h->hy, h->hz, h->gscale64);
        for (int a = 2; a >= 0; --a) fft_axis(h, W, nr, a, +1, s);
        SVH_LAUNCH(k64_gather, blocks_for((int64_t)5 * nr * h->K), 256, 0, s, W, in, out, h->d_vox, h->d_matp,
                   h->d_zloc64, h->K, Nt, 5 * nr, h->kx, h->ky, h->nx, h->ny, (int)green_only);
    }
}

}  // namespace svh
