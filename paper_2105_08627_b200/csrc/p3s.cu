// Plan P3s of the FFT-circulant matvec (SURVEY 8(d) "(H4-H8 fused)"):
// Eq. 9 in THREE HBM passes for thin grids (Nz <= 8, i.e. Kz <= 4):
//
//   A3  x: gather + zero-pad + forward x-FFT of a tile of TY consecutive rows (y) of one
//          non-empty plane, stored TRANSPOSED:  XT = [rc][kx][zp][y]  (zp = index of the
//          non-empty plane, y < Ky), so one kx slab (every y of every non-empty plane) is one
//          contiguous run of Pn*Ky points per component;
//   YZ  per (kx, RHS) slab, on chip: forward y-FFT of the 5 Pn columns (the zero-padded half
//          pruned), then per ky in registers the z-FFT, the 5->5 moment-form MAC with the 7
//          kernel spectra (dense octant or Tucker-expanded, built once per kx into shared
//          memory and reused by every RHS) and the inverse z-FFT, then the inverse y-FFT and
//          the crop to y < Ky -- in place on XT;
//   E3  x: inverse x-FFT + crop + local term z^b I^b + scatter, from TY-row tiles of XT.
//
// Versus P5 (x | y | z | y | x), the 2x-padded y extent and the z pass never leave the chip:
// HBM bytes per RHS ~ 40K + 160 Nx Ry + 80K (Ry = rows of live TY-row blocks of non-empty
// planes) instead of 160 Nx (Rn + Pn Ny) + 120K.  Pruning granularity: a TY-row block of a
// plane holding no voxel is neither written by A3, nor read (zero-filled) / stored by YZ, nor
// read by E3.
//
// FFT structure (all three kernels): N = R1 * R2 two-level Cooley-Tukey with register FFTs
// (reg_fft) of length R1 and R2 and one shared-memory exchange.  In YZ the y spectrum of a
// column stays in shared memory in the two-level order (ky = k1 + R1 k2 at position R2 k1 + k2),
// which every step reads and writes in place (no read/write hazard inside a step).
#include <algorithm>
#include <vector>
#include <cuda_runtime.h>

#include "fft.cuh"
#include "internal.h"
#include "zpass.cuh"   // SpecView, kTuckerMaxRank

namespace svh {
namespace {

__host__ __device__ constexpr int p3_r1(int N) { return 1 << ((ilog2_c(N) + 1) / 2); }
__host__ __device__ constexpr int p3_r2(int N) { return N / p3_r1(N); }

// column / row position p -> padded shared-memory offset (conflict-free strided access)
template <int N>
__device__ __forceinline__ int ppad(int p) { return p + p / p3_r2(N); }
template <int N>
__host__ __device__ constexpr int p3_cs() {   // padded column stride, odd (float2 units)
    return (N + N / p3_r2(N)) | 1;
}
// row tiles of the x passes: element j of row r at r * RS + j + j / R1 (RS odd)
template <int N>
__host__ __device__ constexpr int p3_rs() { return (N + N / p3_r1(N)) | 1; }
template <int N>
__host__ __device__ constexpr int p3_ty() { return N >= 1024 ? 16 : 32; }
template <int N>
__host__ __device__ constexpr int p3_row_nt() { return N >= 512 ? 512 : 256; }

__device__ __forceinline__ int pidx_packed(const int2* __restrict__ rowinfo, int W, int row, int j) {
    const int2 mp = __ldg(&rowinfo[(int64_t)row * W + (j >> 5)]);
    const unsigned bits = (unsigned)mp.x, b = (unsigned)(j & 31);
    return ((bits >> b) & 1u) ? mp.y + __popc(bits & ((1u << b) - 1u)) : -1;
}
__device__ __forceinline__ bool rbit(const uint32_t* __restrict__ rowmask, int rowMW, int z, int y) {
    return (__ldg(&rowmask[(int64_t)z * rowMW + (y >> 5)]) >> (y & 31)) & 1u;
}
// does the TY-row block starting at y0 (a multiple of TY in {16, 32}) of plane z hold a voxel?
__device__ __forceinline__ bool blk_live(const uint32_t* __restrict__ rowmask, int rowMW, int z, int y0, int TY) {
    const uint32_t w = __ldg(&rowmask[(int64_t)z * rowMW + (y0 >> 5)]);
    const uint32_t m = TY >= 32 ? 0xffffffffu : (((1u << TY) - 1u) << (y0 & 31));
    return (w & m) != 0u;
}

struct P3Planes {
    int z_of[8];    // zp -> z
    int zp_of[8];   // z -> zp, or -1 for an empty plane
    int Pn;
};

// ---------------------------------------------------------------------------
// A3: tile = (rc, zp, TY-row block); phase 1 task (row r, n2): R1-point FFT over n1 of
// x[R2 n1 + n2] (the upper half is the zero padding), twiddle W_N^{n2 k1}; phase 2 task
// (r, k1), lanes = rows: R2-point FFT -> kx = k1 + R1 k2, stored to XT (TY consecutive y
// per kx: 128-256-byte runs).
template <int N, bool PACKED>
__global__ void __launch_bounds__(p3_row_nt<N>())
    k_p3_rowA(const float2* __restrict__ in, float2* __restrict__ XT, const int2* __restrict__ rowinfo, int W,
              const uint32_t* __restrict__ rowmask, int rowMW, P3Planes pl, const float2* __restrict__ tw, int Kx,
              int Ky, int64_t K, int64_t Kt, int ntiles, int nyb) {
    constexpr int R1 = p3_r1(N), R2 = p3_r2(N), RS = p3_rs<N>(), TY = p3_ty<N>(), NT = p3_row_nt<N>();
    extern __shared__ float2 S[];   // [TY][RS]
    const float2 zero = make_float2(0.f, 0.f);
    const int Pn = pl.Pn;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int yb = tile % nyb, rest = tile / nyb;
        const int zp = rest % Pn, rc = rest / Pn;
        const int z = pl.z_of[zp], y0 = yb * TY;
        if (!blk_live(rowmask, rowMW, z, y0, TY)) continue;   // CTA-uniform
        __syncthreads();   // the previous tile's phase-2 reads are done
        for (int t = threadIdx.x; t < TY * R2; t += NT) {
            const int n2 = t % R2, r = t / R2, y = y0 + r;
            const int row = z * Ky + y;
            const bool rok = y < Ky && rbit(rowmask, rowMW, z, y);
            float2 v[R1];
#pragma unroll
            for (int n1 = 0; n1 < R1; ++n1) {
                const int j = R2 * n1 + n2;
                v[n1] = zero;
                if (n1 < R1 / 2 && rok && j < Kx) {
                    if (PACKED) {
                        const int idx = pidx_packed(rowinfo, W, row, j);
                        if (idx >= 0) v[n1] = __ldg(&in[(int64_t)rc * K + idx]);
                    } else {
                        v[n1] = __ldg(&in[(int64_t)rc * Kt + (int64_t)row * Kx + j]);
                    }
                }
            }
            reg_fft<R1, -1, true>(v);
#pragma unroll
            for (int k1 = 1; k1 < R1; ++k1) v[k1] = cmul(v[k1], __ldg(&tw[n2 * k1]));
#pragma unroll
            for (int k1 = 0; k1 < R1; ++k1) S[r * RS + n2 * R1 + k1 + n2] = v[k1];
        }
        __syncthreads();
        for (int t = threadIdx.x; t < TY * R1; t += NT) {
            const int r = t % TY, k1 = t / TY, y = y0 + r;
            float2 u[R2];
#pragma unroll
            for (int n2 = 0; n2 < R2; ++n2) u[n2] = S[r * RS + n2 * R1 + k1 + n2];
            reg_fft<R2, -1>(u);
            if (y < Ky) {
                float2* dst = XT + ((int64_t)(rc * (int64_t)N + k1) * Pn + zp) * Ky + y;
                const int64_t step = (int64_t)R1 * Pn * Ky;
#pragma unroll
                for (int k2 = 0; k2 < R2; ++k2) dst[k2 * step] = u[k2];
            }
        }
    }
}

// ---------------------------------------------------------------------------
// E3: tile = (rc, plane, TY-row block) over the non-empty planes (packed output) or every
// plane (grid output: empty tiles are written as zeros).  Phase 1 task (r, n2), lanes =
// rows: R1-point inverse FFT over kx = R2 n1 + n2 read from XT, twiddle; phase 2 task
// (r, k1), lanes = k1: R2-point inverse FFT -> x = k1 + R1 k2 < Kx, local term, scatter.
template <int N, bool PACKED>
__global__ void __launch_bounds__(p3_row_nt<N>())
    k_p3_rowE(const float2* __restrict__ XT, float2* __restrict__ out, const float2* __restrict__ in,
              const int2* __restrict__ rowinfo, int W, const uint32_t* __restrict__ rowmask, int rowMW, P3Planes pl,
              const uint8_t* __restrict__ matp, const float2* __restrict__ zloc, int nzl,
              const float2* __restrict__ tw, int Kx, int Ky, int Kz, int64_t K, int64_t Kt, int green_only,
              int ntiles, int nyb) {
    constexpr int R1 = p3_r1(N), R2 = p3_r2(N), RS = p3_rs<N>(), TY = p3_ty<N>(), NT = p3_row_nt<N>();
    extern __shared__ float2 S[];   // [TY][RS]
    __shared__ float2 zs[5][256];   // z^b per component and material
    for (int m = threadIdx.x; m < 5 * nzl; m += NT) zs[m % 5][m / 5] = zloc[m];
    const float2 zero = make_float2(0.f, 0.f);
    const int Pn = pl.Pn;
    const int nplanes = PACKED ? Pn : Kz;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int yb = tile % nyb, rest = tile / nyb;
        const int pi = rest % nplanes, rc = rest / nplanes;
        const int comp = rc % 5;
        const int z = PACKED ? pl.z_of[pi] : pi;
        const int zp = PACKED ? pi : pl.zp_of[pi];
        const int y0 = yb * TY;
        const bool live = zp >= 0 && blk_live(rowmask, rowMW, z, y0, TY);
        if (!live) {
            if (!PACKED) {   // grid output: zeros for rows without data
                for (int t = threadIdx.x; t < TY * Kx; t += NT) {
                    const int r = t / Kx, j = t % Kx;
                    if (y0 + r < Ky) out[(int64_t)rc * Kt + ((int64_t)z * Ky + y0 + r) * Kx + j] = zero;
                }
            }
            continue;
        }
        __syncthreads();   // zs ready / the previous tile's phase-2 reads are done
        for (int t = threadIdx.x; t < TY * R2; t += NT) {
            const int r = t % TY, n2 = t / TY, y = y0 + r;
            float2 v[R1];
            if (y < Ky) {
                const float2* src = XT + ((int64_t)(rc * (int64_t)N + n2) * Pn + zp) * Ky + y;
                const int64_t step = (int64_t)R2 * Pn * Ky;
#pragma unroll
                for (int n1 = 0; n1 < R1; ++n1) v[n1] = src[n1 * step];
            } else {
#pragma unroll
                for (int n1 = 0; n1 < R1; ++n1) v[n1] = zero;
            }
            reg_fft<R1, +1>(v);
#pragma unroll
            for (int k1 = 1; k1 < R1; ++k1) {
                float2 w = __ldg(&tw[n2 * k1]);
                w.y = -w.y;
                v[k1] = cmul(v[k1], w);
            }
#pragma unroll
            for (int k1 = 0; k1 < R1; ++k1) S[r * RS + n2 * R1 + k1 + n2] = v[k1];
        }
        __syncthreads();
        for (int t = threadIdx.x; t < TY * R1; t += NT) {
            const int k1 = t % R1, r = t / R1, y = y0 + r;
            float2 u[R2];
#pragma unroll
            for (int n2 = 0; n2 < R2; ++n2) u[n2] = S[r * RS + n2 * R1 + k1 + n2];
            reg_fft<R2, +1>(u);
            if (y >= Ky) continue;
            const int row = z * Ky + y;
#pragma unroll
            for (int k2 = 0; k2 < R2 / 2; ++k2) {
                const int j = k1 + R1 * k2;
                if (j >= Kx) continue;
                float2 v = u[k2];
                const int64_t cell = (int64_t)row * Kx + j;
                const int idx = pidx_packed(rowinfo, W, row, j);
                if (idx < 0) {
                    if (!PACKED) out[(int64_t)rc * Kt + cell] = zero;
                    continue;
                }
                if (!green_only) {
                    const float2 zb = zs[comp][__ldg(&matp[idx])];
                    const float2 iv = PACKED ? __ldg(&in[(int64_t)rc * K + idx]) : __ldg(&in[(int64_t)rc * Kt + cell]);
                    v = cadd(v, cmul(zb, iv));
                }
                if (PACKED)
                    out[(int64_t)rc * K + idx] = v;
                else
                    out[(int64_t)rc * Kt + cell] = v;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// YZ: one CTA walks kx = blockIdx.x, blockIdx.x + gridDim.x, ...; per kx it builds the 7
// kernel spectra KV[m][oz][oy] (octant in y and z at the fixed kx, folded with the Green
// prefactor g and the moment-form constants) and then transforms every RHS's slab.
template <int NY, int NZ>
struct P3YZ {
    static constexpr int R1 = p3_r1(NY), R2 = p3_r2(NY), CS = p3_cs<NY>();
    static constexpr int HY = NY / 2 + 1, HZ = NZ / 2 + 1;
    static constexpr int NT = 512;
    // KVG = false: the kx's kernel values are built into shared memory once and reused by
    // every RHS; KVG = true (dense spectra, slab + KV too large): read from the kx-major copy
    // of the octant (h->d_kvt, L2-resident, coalesced along ky) by every z-step
    static size_t smem(int Pn, bool tucker, bool kvg) {
        return (size_t)5 * Pn * CS * sizeof(float2) + (kvg ? 0 : (size_t)7 * HZ * HY * sizeof(float)) +
               (tucker ? (size_t)kTuckerMaxRank * kTuckerMaxRank * sizeof(float) : 0);
    }
};

// kx-major copy of the dense octant spectra: kvt[ox][m][oz][oy] = spec[m][oz][oy][ox]
__global__ void k_p3_kvt(const float* __restrict__ spec, float* __restrict__ kvt, int hx, int hy, int hz) {
    const int64_t n = (int64_t)7 * hx * hy * hz;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int oy = (int)(i % hy);
        int64_t r = i / hy;
        const int oz = (int)(r % hz);
        r /= hz;
        const int m = (int)(r % 7);
        const int ox = (int)(r / 7);
        kvt[i] = __ldg(&spec[(((int64_t)m * hz + oz) * hy + oy) * hx + ox]);
    }
}

template <int NY, int NZ, bool KVG>
__global__ void __launch_bounds__(512, 1)
    k_p3_yz(float2* __restrict__ XT, SpecView sv, const float* __restrict__ kvt, const float2* __restrict__ tw,
            int Nx, int Ky, int Kz, const uint32_t* __restrict__ rowmask, int rowMW, P3Planes pl, int TY, float g,
            int nrhs) {
    using P = P3YZ<NY, NZ>;
    constexpr int R1 = P::R1, R2 = P::R2, CS = P::CS, HY = P::HY, HZ = P::HZ, NT = P::NT;
    constexpr int NZH = NZ / 2;
    constexpr int NZL = NZ == 1 ? 1 : NZH;   // planes that can hold voxels (Kz <= NZL)
    extern __shared__ float2 S[];                                   // [5 Pn][CS]
    const int Pn = pl.Pn;
    float* KV = reinterpret_cast<float*>(S + 5 * Pn * CS);         // [7][HZ][HY]
    float* A = KV + 7 * HZ * HY;                                    // Tucker scratch [d3][d2]
    __shared__ uint64_t live[8];                                    // TY-row block liveness per zp
    const int tid = threadIdx.x;
    const float2 zero = make_float2(0.f, 0.f);
    const int nyb = (Ky + TY - 1) / TY;
    if (tid < Pn) {
        int z = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if (i == tid) z = pl.z_of[i];   // constant-index param reads (no local copy)
        uint64_t m = 0;
        for (int b = 0; b < nyb; ++b)
            if (blk_live(rowmask, rowMW, z, b * TY, TY)) m |= 1ull << b;
        live[tid] = m;
    }
    const int lg_ty = TY == 16 ? 4 : 5;
    const int64_t slab = (int64_t)Pn * Ky;                          // points per (rc, kx)
    for (int kx = blockIdx.x; kx < Nx; kx += gridDim.x) {
        const int ox = kx <= (Nx >> 1) ? kx : Nx - kx;
        const float sx = kx <= (Nx >> 1) ? 1.f : -1.f;
        // moment-form constants folded into the kernel values (k_zmac2): m = 1 carries sx,
        // m = 3 carries -2, m = 6 carries 4 (K1y's sy and K1z's kz sign are applied per point)
        auto fold = [&](int m) -> float { return m == 1 ? g * sx : m == 3 ? -2.f * g : m == 6 ? 4.f * g : g; };
        __syncthreads();   // the previous kx's last z-step reads of KV are done
        const float* KVp = KVG ? kvt + (int64_t)ox * 7 * HZ * HY : KV;
        // in KVG mode the folds are applied per point (the table holds raw spectra)
        const float c0 = KVG ? g : 1.f, c1 = KVG ? g * sx : 1.f, c3 = KVG ? -2.f * g : 1.f, c6 = KVG ? 4.f * g : 1.f;
        if (KVG) {
        } else if (sv.spec) {
            const int64_t plo = (int64_t)sv.hx * sv.hy * sv.hz;
            for (int t = tid; t < 7 * HZ * HY; t += NT) {
                const int m = t / (HZ * HY), rem = t % (HZ * HY);
                const int oz = rem / HY, oy = rem % HY;
                KV[t] = __ldg(&sv.spec[m * plo + ((int64_t)oz * sv.hy + oy) * sv.hx + ox]) * fold(m);
            }
        } else {
            // Tucker (Eq. 10): KV[m](oy, oz) = sum_c3 F3[oz][c3] sum_c2 F2[oy][c2] A[c3][c2],
            // A[c3][c2] = sum_c1 core[c3][c2][c1] F1[ox][c1]
            for (int m = 0; m < 7; ++m) {
                const int d1 = sv.rk[m][0], d2 = sv.rk[m][1], d3 = sv.rk[m][2];
                const float* C = sv.core[m];
                const float* f1 = sv.fac[m][0] + (int64_t)ox * d1;
                for (int t = tid; t < d3 * d2; t += NT) {
                    float acc = 0.f;
                    for (int c1 = 0; c1 < d1; ++c1) acc = fmaf(__ldg(&C[(int64_t)t * d1 + c1]), __ldg(&f1[c1]), acc);
                    A[t] = acc;
                }
                __syncthreads();
                const float* F2 = sv.fac[m][1];
                const float* F3 = sv.fac[m][2];
                for (int oy = tid; oy < HY; oy += NT) {
                    float B[kTuckerMaxRank];
#pragma unroll
                    for (int c3 = 0; c3 < kTuckerMaxRank; ++c3) {
                        float acc = 0.f;
                        if (c3 < d3)
                            for (int c2 = 0; c2 < d2; ++c2) acc = fmaf(A[c3 * d2 + c2], __ldg(&F2[(int64_t)oy * d2 + c2]), acc);
                        B[c3] = acc;
                    }
#pragma unroll
                    for (int oz = 0; oz < HZ; ++oz) {
                        float acc = 0.f;
#pragma unroll
                        for (int c3 = 0; c3 < kTuckerMaxRank; ++c3)
                            if (c3 < d3) acc = fmaf(B[c3], __ldg(&F3[oz * d3 + c3]), acc);
                        KV[(m * HZ + oz) * HY + oy] = acc * fold(m);
                    }
                }
                __syncthreads();
            }
        }
        for (int r = 0; r < nrhs; ++r) {
            float2* base = XT + ((int64_t)r * 5 * Nx + kx) * slab;   // component c at + c * Nx * slab
            const int64_t cstride = (int64_t)Nx * slab;
            // the next slab (this kx's next RHS, or the next kx's first) -> L2
            if (tid < 5) {
                const float2* nb = nullptr;
                if (r + 1 < nrhs)
                    nb = base + 5 * cstride + tid * cstride;
                else if (kx + (int)gridDim.x < Nx)
                    nb = XT + (kx + gridDim.x) * slab + tid * cstride;
                const uint32_t bytes = (uint32_t)(slab * 8) & ~15u;
                if (nb && bytes && (((uintptr_t)nb) & 15u) == 0)
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(nb), "r"(bytes) : "memory");
            }
            __syncthreads();   // KV built / the previous slab's inverse phase-2 reads are done
            // forward y, phase 1: task (col, n2): x[R2 n1 + n2], n1 < R1/2 (rows >= Ky and rows
            // of dead blocks are zero) -> Y[n2][k1] W^{n2 k1} at position R2 k1 + n2
            for (int t = tid; t < 5 * Pn * R2; t += NT) {
                const int n2 = t % R2, col = t / R2;
                const int c = col / Pn, zp = col % Pn;
                const float2* src = base + c * cstride + (int64_t)zp * Ky;
                const uint64_t lm = live[zp];
                float2 v[R1];
#pragma unroll
                for (int n1 = 0; n1 < R1; ++n1) {
                    const int y = R2 * n1 + n2;
                    v[n1] = (n1 < R1 / 2 && y < Ky && ((lm >> (y >> lg_ty)) & 1ull)) ? src[y] : zero;
                }
                reg_fft<R1, -1, true>(v);
                float2* Sc = S + col * CS;
#pragma unroll
                for (int k1 = 0; k1 < R1; ++k1) {
                    const float2 w = k1 ? __ldg(&tw[n2 * k1]) : make_float2(1.f, 0.f);
                    Sc[ppad<NY>(R2 * k1 + n2)] = k1 ? cmul(v[k1], w) : v[k1];
                }
            }
            __syncthreads();
            // forward y, phase 2: task (col, k1): R2-point FFT of the block R2 k1 + n2, in place
            for (int t = tid; t < 5 * Pn * R1; t += NT) {
                const int k1 = t % R1, col = t / R1;
                float2* Sc = S + col * CS + k1 * (R2 + 1);
                float2 u[R2];
#pragma unroll
                for (int n2 = 0; n2 < R2; ++n2) u[n2] = Sc[n2];
                reg_fft<R2, -1>(u);
#pragma unroll
                for (int k2 = 0; k2 < R2; ++k2) Sc[k2] = u[k2];
            }
            __syncthreads();
            // z-step per ky (position R2 (ky % R1) + ky / R1): z-FFT, MAC, inverse z-FFT
            for (int ky = tid; ky < NY; ky += NT) {
                const int pos = ppad<NY>(R2 * (ky % R1) + ky / R1);
                const int oy = ky <= (NY >> 1) ? ky : NY - ky;
                const float sy = ky <= (NY >> 1) ? 1.f : -1.f;
                float2 v[5][NZ];
#pragma unroll
                for (int c = 0; c < 5; ++c)
#pragma unroll
                    for (int z = 0; z < NZ; ++z) {
                        const int zp = z < NZL && z < Kz ? pl.zp_of[z] : -1;
                        v[c][z] = zp >= 0 ? S[(c * Pn + zp) * CS + pos] : zero;
                    }
#pragma unroll
                for (int c = 0; c < 5; ++c) reg_fft<NZ, -1, (NZ > 1)>(v[c]);
#pragma unroll
                for (int k = 0; k < NZ; ++k) {
                    const int oz = k <= NZH ? k : NZ - k;
                    const float s3 = k <= NZH ? 1.f : -1.f;   // K1z is odd in kz
                    const float* kp = KVp + oz * HY + oy;
                    float kk[7];
#pragma unroll
                    for (int m = 0; m < 7; ++m) kk[m] = KVG ? __ldg(&kp[m * HZ * HY]) : kp[m * HZ * HY];
                    const float f0 = c0 * kk[0], f1 = c1 * kk[1], f2 = (c0 * sy) * kk[2];
                    const float f3 = (c3 * s3) * kk[3], f4 = c0 * kk[4], f5 = c0 * kk[5];
                    const float f6 = c6 * kk[6];
                    const float2 Ix = v[0][k], Iy = v[1][k], Iz = v[2][k], I2 = v[3][k], I3 = v[4][k];
                    const float2 m1x = cadd(I2, I3), m1y = csub(I3, I2);
                    const float2 Qx = cfma_s(Ix, -f1, cmul_i(m1x, f4));
                    const float2 Qy = cfma_s(Iy, -f2, cmul_i(m1y, f5));
                    const float2 Qz = cfma_s(Iz, -f3, cmul_i(I3, f6));
                    v[0][k] = cfma_s(m1x, f1, cmul_i(Ix, f0));
                    v[1][k] = cfma_s(m1y, f2, cmul_i(Iy, f0));
                    v[2][k] = cfma_s(I3, f3, cmul_i(Iz, f0));
                    v[3][k] = csub(Qx, Qy);
                    v[4][k] = cadd(cadd(Qx, Qy), Qz);
                }
#pragma unroll
                for (int c = 0; c < 5; ++c) reg_fft<NZ, +1>(v[c]);
#pragma unroll
                for (int c = 0; c < 5; ++c)
#pragma unroll
                    for (int z = 0; z < NZL; ++z) {
                        const int zp = z < Kz ? pl.zp_of[z] : -1;
                        if (zp >= 0) S[(c * Pn + zp) * CS + pos] = v[c][z];
                    }
            }
            __syncthreads();
            // inverse y, phase 1: task (col, k1): R2-point inverse FFT over k2 of the block
            // R2 k1 + k2, twiddle W^{-n2 k1}, in place (position R2 k1 + n2)
            for (int t = tid; t < 5 * Pn * R1; t += NT) {
                const int k1 = t % R1, col = t / R1;
                float2* Sc = S + col * CS + k1 * (R2 + 1);
                float2 u[R2];
#pragma unroll
                for (int k2 = 0; k2 < R2; ++k2) u[k2] = Sc[k2];
                reg_fft<R2, +1>(u);
#pragma unroll
                for (int n2 = 0; n2 < R2; ++n2) {
                    if (n2 && k1) {
                        float2 w = __ldg(&tw[n2 * k1]);
                        w.y = -w.y;
                        u[n2] = cmul(u[n2], w);
                    }
                    Sc[n2] = u[n2];
                }
            }
            __syncthreads();
            // inverse y, phase 2: task (col, n2): R1-point inverse FFT over k1 -> y = R2 n1 + n2,
            // the kept y < Ky of live blocks stored to XT
            for (int t = tid; t < 5 * Pn * R2; t += NT) {
                const int n2 = t % R2, col = t / R2;
                const int c = col / Pn, zp = col % Pn;
                const float2* Sc = S + col * CS;
                float2 v[R1];
#pragma unroll
                for (int k1 = 0; k1 < R1; ++k1) v[k1] = Sc[ppad<NY>(R2 * k1 + n2)];
                reg_fft<R1, +1>(v);
                float2* dst = base + c * cstride + (int64_t)zp * Ky;
                const uint64_t lm = live[zp];
#pragma unroll
                for (int n1 = 0; n1 < R1 / 2; ++n1) {
                    const int y = R2 * n1 + n2;
                    if (y < Ky && ((lm >> (y >> lg_ty)) & 1ull)) dst[y] = v[n1];
                }
            }
        }
    }
}

// kernel attributes and resident-CTA counts are queried once per (device, kernel, size): these
// driver calls cost host time on every launch otherwise, and a P3s product on a thin grid is
// only ~0.5 ms of device work
struct AttrRec {
    int dev;
    const void* k;
    size_t smem;
    int ctas;
};
template <typename F>
int grid_for(F* kern, int nt, size_t smem, int64_t units) {
    static thread_local std::vector<AttrRec> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    int ctas = 0;
    for (const auto& r : cache)
        if (r.dev == dev && r.k == (const void*)kern && r.smem == smem) ctas = r.ctas;
    if (ctas == 0) {
        SVH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                      (int)cudaSharedmemCarveoutMaxShared));
        // the attribute is sticky per kernel: never lower it below a size cached earlier
        size_t top = smem;
        for (const auto& r : cache)
            if (r.dev == dev && r.k == (const void*)kern) top = std::max(top, r.smem);
        SVH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)top));
        int nsm = 148, occ = 1;
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, nt, smem);
        ctas = nsm * std::max(occ, 1);
        cache.push_back(AttrRec{dev, (const void*)kern, smem, ctas});
    }
    return (int)std::max<int64_t>(1, std::min<int64_t>(units, ctas));
}

P3Planes planes_of(const svh_handle* h) {
    P3Planes pl{};
    for (int z = 0; z < 8; ++z) pl.zp_of[z] = -1, pl.z_of[z] = 0;
    int n = 0;
    for (int z = 0; z < h->kz && z < 8; ++z)
        if ((h->planemask >> z) & 1ull) {
            pl.z_of[n] = z;
            pl.zp_of[z] = n++;
        }
    pl.Pn = n;
    return pl;
}

bool tucker_fits(const svh_handle* h) {
    if (!h->use_tucker) return true;
    for (int m = 0; m < 7; ++m)
        for (int a = 0; a < 3; ++a)
            if (h->tucker.ranks[m][a] > kTuckerMaxRank) return false;
    return true;
}

constexpr size_t kSmemMax = 227 * 1024;

// 0 = not eligible, 1 = kernel values in shared memory, 2 = kernel values from d_kvt
template <int NY, int NZ>
int yz_mode(const svh_handle* h) {
    const int Pn = planes_of(h).Pn;
    if (P3YZ<NY, NZ>::smem(Pn, h->use_tucker, false) <= kSmemMax) return 1;
    if (!h->use_tucker && P3YZ<NY, NZ>::smem(Pn, false, true) <= kSmemMax) return 2;
    return 0;
}

#define P3_DISPATCH_X(n, CALL)                        \
    switch (n) {                                      \
        case 128: { constexpr int NX = 128; CALL; break; }   \
        case 256: { constexpr int NX = 256; CALL; break; }   \
        case 512: { constexpr int NX = 512; CALL; break; }   \
        case 1024: { constexpr int NX = 1024; CALL; break; } \
        default: throw Error{SVH_EINVAL, "P3s: x extent"};   \
    }
#define P3_DISPATCH_Y(n, CALL)                        \
    switch (n) {                                      \
        case 8: { constexpr int NY = 8; CALL; break; }       \
        case 16: { constexpr int NY = 16; CALL; break; }     \
        case 32: { constexpr int NY = 32; CALL; break; }     \
        case 64: { constexpr int NY = 64; CALL; break; }     \
        case 128: { constexpr int NY = 128; CALL; break; }   \
        case 256: { constexpr int NY = 256; CALL; break; }   \
        case 512: { constexpr int NY = 512; CALL; break; }   \
        case 1024: { constexpr int NY = 1024; CALL; break; } \
        default: throw Error{SVH_EINVAL, "P3s: y extent"};   \
    }
#define P3_DISPATCH_Z(n, CALL)                        \
    switch (n) {                                      \
        case 1: { constexpr int NZ = 1; CALL; break; }       \
        case 2: { constexpr int NZ = 2; CALL; break; }       \
        case 4: { constexpr int NZ = 4; CALL; break; }       \
        case 8: { constexpr int NZ = 8; CALL; break; }       \
        default: throw Error{SVH_EINVAL, "P3s: z extent"};   \
    }

template <int NX>
void run_a3(svh_handle* h, const P3Planes& pl, const float2* in, float2* XT, bool packed, int nr, cudaStream_t s) {
    constexpr int TY = p3_ty<NX>(), NT = p3_row_nt<NX>();
    const int nyb = (h->ky + TY - 1) / TY;
    const int64_t ntiles = (int64_t)5 * nr * pl.Pn * nyb;
    const size_t smem = (size_t)TY * p3_rs<NX>() * sizeof(float2);
    auto go = [&](auto kern) {
        SVH_LAUNCH(kern, grid_for(kern, NT, smem, ntiles), NT, smem, s, in, XT, h->d_rowinfo, h->rowW, h->d_rowmask,
                   h->rowMW, pl, h->d_tw[0], h->kx, h->ky, h->K, h->Kt, (int)ntiles, nyb);
    };
    if (packed)
        go(k_p3_rowA<NX, true>);
    else
        go(k_p3_rowA<NX, false>);
}

template <int NX>
void run_e3(svh_handle* h, const P3Planes& pl, const float2* XT, const float2* in, float2* out, bool packed,
            bool green_only, int nr, cudaStream_t s) {
    constexpr int TY = p3_ty<NX>(), NT = p3_row_nt<NX>();
    const int nyb = (h->ky + TY - 1) / TY;
    const int64_t ntiles = (int64_t)5 * nr * (packed ? pl.Pn : h->kz) * nyb;
    const size_t smem = (size_t)TY * p3_rs<NX>() * sizeof(float2);
    const int nzl = (int)h->mats.size() + 1;
    auto go = [&](auto kern) {
        SVH_LAUNCH(kern, grid_for(kern, NT, smem, ntiles), NT, smem, s, XT, out, in, h->d_rowinfo, h->rowW,
                   h->d_rowmask, h->rowMW, pl, h->d_matp, h->d_zloc, nzl, h->d_tw[0], h->kx, h->ky, h->kz, h->K,
                   h->Kt, (int)green_only, (int)ntiles, nyb);
    };
    if (packed)
        go(k_p3_rowE<NX, true>);
    else
        go(k_p3_rowE<NX, false>);
}

template <int NY, int NZ>
void run_yz(svh_handle* h, const P3Planes& pl, float2* XT, int TY, int nr, cudaStream_t s) {
    SpecView sv{};
    sv.spec = h->use_tucker ? nullptr : h->d_spec;
    sv.hx = h->hx;
    sv.hy = h->hy;
    sv.hz = h->hz;
    if (h->use_tucker)
        for (int m = 0; m < 7; ++m) {
            sv.core[m] = h->tucker.d_core[m];
            for (int a = 0; a < 3; ++a) {
                sv.fac[m][a] = h->tucker.d_factor[m][a];
                sv.rk[m][a] = h->tucker.ranks[m][a];
            }
        }
    const int mode = yz_mode<NY, NZ>(h);
    SVH_CHECK(mode > 0, SVH_EINVAL, "P3s: y-z slab does not fit shared memory");
    if (mode == 2 && !h->d_kvt) {
        const int64_t n = (int64_t)7 * h->hx * h->hy * h->hz;
        SVH_CUDA(cudaMalloc(&h->d_kvt, n * sizeof(float)));
        SVH_LAUNCH(k_p3_kvt, (int)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, s, h->d_spec, h->d_kvt, h->hx,
                   h->hy, h->hz);
    }
    auto go = [&](auto kern, bool kvg) {
        const size_t smem = P3YZ<NY, NZ>::smem(pl.Pn, h->use_tucker, kvg);
        SVH_LAUNCH(kern, grid_for(kern, 512, smem, h->nx), 512, smem, s, XT, sv, h->d_kvt, h->d_tw[1], h->nx, h->ky,
                   h->kz, h->d_rowmask, h->rowMW, pl, TY, h->gscale, nr);
    };
    if (mode == 2)
        go(k_p3_yz<NY, NZ, true>, true);
    else
        go(k_p3_yz<NY, NZ, false>, false);
}

}  // namespace

bool p3s_eligible(const svh_handle* h) {
    if (h->nz != 1 && h->nz != 2 && h->nz != 4 && h->nz != 8) return false;
    if (h->nx < 128 || h->nx > 1024) return false;
    if (h->ny < 8 || h->ny > 1024) return false;
    if (h->kz > 8 || h->nzp < 1 || !tucker_fits(h)) return false;
    int mode = 0;
    P3_DISPATCH_Y(h->ny, P3_DISPATCH_Z(h->nz, (mode = yz_mode<NY, NZ>(h))));
    return mode > 0;
}

// one sub-batch of nr RHS (XT = the X1 workspace slice: nr x 5 x Nx x Pn x Ky points)
void p3s_matvec(svh_handle* h, const float2* in, float2* out, float2* XT, int nr, bool green_only, bool packed,
                cudaStream_t s) {
    const P3Planes pl = planes_of(h);
    int TY = 32;
    P3_DISPATCH_X(h->nx, (TY = p3_ty<NX>()));
    P3_DISPATCH_X(h->nx, run_a3<NX>(h, pl, in, XT, packed, nr, s));
    P3_DISPATCH_Y(h->ny, P3_DISPATCH_Z(h->nz, (run_yz<NY, NZ>(h, pl, XT, TY, nr, s))));
    P3_DISPATCH_X(h->nx, run_e3<NX>(h, pl, XT, in, out, packed, green_only, nr, s));
}

}  // namespace svh
