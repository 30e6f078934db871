// FFT-circulant VIE matvec, Eq. 9:
//   CC^b = z^b I^b + IFFT{ sum_a Zhat^{b,a} * FFT(I^a) }   (cropped to the voxels)
//
// Plan P5: five passes over HBM per right-hand side,
//   A  x: gather from packed order + zero-pad + forward FFT along x          Kt -> 2Kt pts/comp
//   B  y: zero-pad + forward FFT along y (strided pencils)                    2Kt -> 4Kt
//   C  z: zero-pad + forward FFT along z, 5->5 moment-form MAC with the 7
//         kernel spectra, inverse FFT, crop (in place)                        4Kt -> 4Kt
//   D  y: inverse FFT along y + crop                                          4Kt -> 2Kt
//   E  x: inverse FFT along x + crop + local term z^b I^b + scatter to packed 2Kt -> Kt
// Layouts: X1 = [rhs][5][Kz][Ky][Nx], X2 = [rhs][5][Kz][Ny][Nx] (complex64).
//
// FFT structure (fft.cuh): lengths N <= 64 run entirely in one thread's
// registers; longer ones use N = R1*R2 with the first R1-point FFTs loaded
// straight from global memory into registers, one shared-memory transpose,
// and the R2-point FFTs stored straight from registers to global memory.
// Zero padding (forward: upper half of the input is zero) and cropping
// (inverse: only the lower half of the output is kept) are compile-time
// prunings of the first / last stage.
#include <algorithm>
#include <cstdlib>
#include <string>
#include <cuda_runtime.h>

#include "fft.cuh"
#include "internal.h"
#include "rowfft.cuh"
#include "zpass.cuh"
#include "ypass.cuh"
#include "tma.cuh"

namespace svh {

// ---------------------------------------------------------------------------
// shared-memory index helpers (bank-conflict padding)
// "pencil-major" layout for passes A/E: element j of row q at q*(N + N/R1) + j + j/R1
template <int N>
__device__ __forceinline__ int pm_idx(int q, int j) {
    constexpr int R1 = fft_r1(N);
    return q * (N + N / R1) + j + j / R1;
}
// "element-major" layout for strided passes: element j of pencil q at j*Q + q, plus Q
// per R1-block when Q < 16 (so the 32/Q pencil-rows a warp stores hit distinct banks)
template <int N, int Q>
__device__ __forceinline__ int em_idx(int j, int q) {
    constexpr int R1 = fft_r1(N);
    return j * Q + q + (Q < 16 ? (j / R1) * Q : 0);
}
template <int N, int Q>
constexpr int em_size() {
    return N * Q + (Q < 16 ? (N / fft_r1(N)) * Q : 0);
}

// ---------------------------------------------------------------------------
// Row passes A (forward, gather + pad) and E (inverse, crop + local term + scatter).
// Row length N along x, Q rows per CTA; threads = TPP*Q with TPP = threads per pencil.
// Row occupancy words (rowinfo[row][j/32] = {bits, packed index of the word's first voxel})
// give the packed index of voxel j of a row as pre + popc(bits below j): one tiny,
// L1-resident load instead of a Kt-sized index map.
__device__ __forceinline__ int packed_index(const int2* __restrict__ rowinfo, int W, int row, int j) {
    const int2 mp = __ldg(&rowinfo[(int64_t)row * W + (j >> 5)]);
    const unsigned bits = (unsigned)mp.x, b = (unsigned)(j & 31);
    return ((bits >> b) & 1u) ? mp.y + __popc(bits & ((1u << b) - 1u)) : -1;
}

// row_bit: does row (y, z) of the lattice hold a voxel?  (rows that do not are zero in
// every embedded current; the passes neither write nor read them)
__device__ __forceinline__ bool row_bit(const uint32_t* __restrict__ rowmask, int rowMW, int z, int y) {
    return (__ldg(&rowmask[(int64_t)z * rowMW + (y >> 5)]) >> (y & 31)) & 1u;
}

// Pass A over the non-empty rows only (rowlist[li], li < nlist, global row z*Ky + y); X1
// keeps the [rc][rows][N] layout so the strided passes index it by (z, y).  A y-slab
// (rows y0 <= y < y0 + Kyl of every plane) uses the local row
// z*Kyl + y - y0 for X1 and for a grid-layout input; the whole grid is Kyl = Ky, y0 = 0.
template <int N, int Q, bool PACKED>
__global__ void __launch_bounds__(fft_threads_per_pencil(N) * Q)
    k_row_fwd(const float2* __restrict__ in, float2* __restrict__ X1, const int2* __restrict__ rowinfo, int W,
              const int32_t* __restrict__ rowlist, int nlist, const float2* __restrict__ tw, int Kx, int rows,
              int64_t K, int64_t Kt, int Ky, int Kyl, int y0) {
    constexpr int R1 = fft_r1(N), R2 = fft_r2(N);
    const int rc = blockIdx.y;
    const int li0 = blockIdx.x * Q;
    const float2 zero = make_float2(0.f, 0.f);
    auto row_of = [&](int q) -> int { return li0 + q < nlist ? __ldg(&rowlist[li0 + q]) : -1; };
    auto local = [&](int row) -> int { return (row / Ky) * Kyl + row % Ky - y0; };
    auto load = [&](int row, int j) -> float2 {
        if (row < 0 || j >= Kx) return zero;
        const int idx = packed_index(rowinfo, W, row, j);
        if (idx < 0) return zero;
        return PACKED ? __ldg(&in[(int64_t)rc * K + idx])
                      : __ldg(&in[(int64_t)rc * Kt + (int64_t)local(row) * Kx + j]);
    };
    if constexpr (R2 == 1) {
        const int row = row_of(threadIdx.x);
        float2 v[N];
#pragma unroll
        for (int j = 0; j < N; ++j) v[j] = (j < N / 2 || N == 1) ? load(row, j) : zero;
        reg_fft<N, -1, (N > 1)>(v);
        if (row >= 0) {
            float2* dst = X1 + ((int64_t)rc * rows + local(row)) * N;
#pragma unroll
            for (int k = 0; k < N; ++k) dst[k] = v[k];
        }
    } else {
        extern __shared__ float2 S[];
        if (threadIdx.x < R2 * Q) {
            const int q = threadIdx.x / R2, n2 = threadIdx.x % R2;
            const int row = row_of(q);
            float2 v[R1];
#pragma unroll
            for (int n1 = 0; n1 < R1; ++n1) v[n1] = (n1 < R1 / 2) ? load(row, R2 * n1 + n2) : zero;
            reg_fft<R1, -1, true>(v);
#pragma unroll
            for (int k1 = 1; k1 < R1; ++k1) v[k1] = cmul(v[k1], __ldg(&tw[n2 * k1]));
#pragma unroll
            for (int k1 = 0; k1 < R1; ++k1) S[pm_idx<N>(q, n2 * R1 + k1)] = v[k1];
        }
        __syncthreads();
        if (threadIdx.x < R1 * Q) {
            const int q = threadIdx.x / R1, k1 = threadIdx.x % R1;
            const int row = row_of(q);
            float2 u[R2];
#pragma unroll
            for (int n2 = 0; n2 < R2; ++n2) u[n2] = S[pm_idx<N>(q, n2 * R1 + k1)];
            reg_fft<R2, -1>(u);
            if (row >= 0) {
                float2* dst = X1 + ((int64_t)rc * rows + local(row)) * N;
#pragma unroll
                for (int k2 = 0; k2 < R2; ++k2) dst[k1 + R1 * k2] = u[k2];
            }
        }
    }
}

// Pass E over the rows rowlist[li] (packed output: the non-empty rows) or over all
// rows (rowlist == nullptr, grid output: empty rows are written as zeros without
// reading X1, which holds no data for them).
template <int N, int Q, bool PACKED>
__global__ void __launch_bounds__(fft_threads_per_pencil(N) * Q)
    k_row_inv(const float2* __restrict__ X1, float2* __restrict__ out, const float2* __restrict__ in,
              const int2* __restrict__ rowinfo, int W, const int32_t* __restrict__ rowlist, int nlist,
              const uint32_t* __restrict__ rowmask, int rowMW, int Ky, const uint8_t* __restrict__ matp,
              const float2* __restrict__ zloc, int nzl, const float2* __restrict__ tw, int Kx, int rows, int64_t K,
              int64_t Kt, int green_only, int Kyl, int y0) {
    constexpr int R1 = fft_r1(N), R2 = fft_r2(N);
    const int rc = blockIdx.y;
    const int comp = rc % 5;
    const int li0 = blockIdx.x * Q;
    const float2 zero = make_float2(0.f, 0.f);
    __shared__ float2 zs[256];   // z^b of this component per material
    for (int m = threadIdx.x; m < nzl; m += blockDim.x) zs[m] = zloc[m * 5 + comp];
    __syncthreads();
    // global row z*Ky + y of slot q (rowlist: packed output over the non-empty rows;
    // nullptr: every row of the (slab) grid, local slot z*Kyl + y - y0)
    auto row_of = [&](int q) -> int {
        const int li = li0 + q;
        if (li >= nlist) return -1;
        return rowlist ? __ldg(&rowlist[li]) : (li / Kyl) * Ky + y0 + li % Kyl;
    };
    auto local = [&](int row) -> int { return (row / Ky) * Kyl + row % Ky - y0; };
    // X1 holds data for this row (listed rows are non-empty by construction)
    auto live = [&](int row) -> bool {
        return row >= 0 && (rowlist != nullptr || row_bit(rowmask, rowMW, row / Ky, row % Ky));
    };
    auto store = [&](int row, int j, float2 v) {
        if (row < 0 || j >= Kx) return;
        const int64_t cell = (int64_t)local(row) * Kx + j;
        const int idx = packed_index(rowinfo, W, row, j);
        if (idx < 0) {
            if (!PACKED) out[(int64_t)rc * Kt + cell] = zero;
            return;
        }
        if (!green_only) {
            const float2 z = zs[__ldg(&matp[idx])];
            const float2 iv = PACKED ? __ldg(&in[(int64_t)rc * K + idx]) : __ldg(&in[(int64_t)rc * Kt + cell]);
            v = cadd(v, cmul(z, iv));
        }
        if (PACKED)
            out[(int64_t)rc * K + idx] = v;
        else
            out[(int64_t)rc * Kt + cell] = v;
    };
    if constexpr (R2 == 1) {
        const int row = row_of(threadIdx.x);
        const bool ok = live(row);
        float2 v[N];
        const float2* src = X1 + ((int64_t)rc * rows + (ok ? local(row) : 0)) * N;
#pragma unroll
        for (int k = 0; k < N; ++k) v[k] = ok ? src[k] : zero;
        reg_fft<N, +1>(v);
#pragma unroll
        for (int j = 0; j < (N + 1) / 2; ++j) store(row, j, v[j]);
    } else {
        extern __shared__ float2 S[];
        if (threadIdx.x < R2 * Q) {
            const int q = threadIdx.x / R2, n2 = threadIdx.x % R2;
            const int row = row_of(q);
            const bool ok = live(row);
            const float2* src = X1 + ((int64_t)rc * rows + (ok ? local(row) : 0)) * N;
            float2 v[R1];
#pragma unroll
            for (int n1 = 0; n1 < R1; ++n1) v[n1] = ok ? src[R2 * n1 + n2] : zero;
            reg_fft<R1, +1>(v);
#pragma unroll
            for (int k1 = 1; k1 < R1; ++k1) {
                float2 w = __ldg(&tw[n2 * k1]);
                w.y = -w.y;
                v[k1] = cmul(v[k1], w);
            }
#pragma unroll
            for (int k1 = 0; k1 < R1; ++k1) S[pm_idx<N>(q, n2 * R1 + k1)] = v[k1];
        }
        __syncthreads();
        if (threadIdx.x < R1 * Q) {
            const int q = threadIdx.x / R1, k1 = threadIdx.x % R1;
            const int row = row_of(q);
            float2 u[R2];
#pragma unroll
            for (int n2 = 0; n2 < R2; ++n2) u[n2] = S[pm_idx<N>(q, n2 * R1 + k1)];
            reg_fft<R2, +1>(u);
#pragma unroll
            for (int k2 = 0; k2 < R2 / 2; ++k2) store(row, k1 + R1 * k2, u[k2]);
        }
    }
}

// ---------------------------------------------------------------------------
// Strided passes B / D (pencils along y, stride Nx).  Tile = Q consecutive kx at one
// non-empty plane z = planes[blockIdx.y] and one (rhs, component).
// DIR = -1: input rows j < Lin (<= N/2), zero-padded, and only rows (j, z) holding a
//           voxel are read (the others are zero and were never written by pass A); all N outputs.
// DIR = +1: all N inputs; outputs j < Lout (<= N/2) of the rows pass E reads.
template <int N, int Q, int DIR>
__global__ void __launch_bounds__(fft_threads_per_pencil(N) * Q)
    k_col(const float2* __restrict__ in, float2* __restrict__ out, const float2* __restrict__ tw, int Nx, int Kz,
          int Lin, int Lout, const int32_t* __restrict__ planes, const uint32_t* __restrict__ rowmask, int rowMW) {
    constexpr int R1 = fft_r1(N), R2 = fft_r2(N);
    const int kx0 = blockIdx.x * Q;
    const int z = __ldg(&planes[blockIdx.y]);
    const int64_t rc = blockIdx.z;
    const float2* src = in + ((rc * Kz + z) * Lin) * (int64_t)Nx + kx0;
    float2* dst = out + ((rc * Kz + z) * Lout) * (int64_t)Nx + kx0;
    const float2 zero = make_float2(0.f, 0.f);
    auto live = [&](int j) { return row_bit(rowmask, rowMW, z, j); };
    if constexpr (R2 == 1) {
        const int q = threadIdx.x;
        if (kx0 + q >= Nx) return;
        float2 v[N];
#pragma unroll
        for (int j = 0; j < N; ++j) {
            if (DIR < 0)
                v[j] = ((j < N / 2 || N == 1) && j < Lin && live(j)) ? src[(int64_t)j * Nx + q] : zero;
            else
                v[j] = src[(int64_t)j * Nx + q];
        }
        reg_fft<N, DIR>(v);
#pragma unroll
        for (int j = 0; j < N; ++j) {
            if (DIR < 0 || (j < (N + 1) / 2 && j < Lout && live(j))) dst[(int64_t)j * Nx + q] = v[j];
        }
    } else {
        extern __shared__ float2 S[];
        if (threadIdx.x < R2 * Q) {
            const int n2 = threadIdx.x / Q, q = threadIdx.x % Q;
            const bool ok = kx0 + q < Nx;
            float2 v[R1];
#pragma unroll
            for (int n1 = 0; n1 < R1; ++n1) {
                const int j = R2 * n1 + n2;
                if (DIR < 0)
                    v[n1] = (n1 < R1 / 2 && j < Lin && ok && live(j)) ? src[(int64_t)j * Nx + q] : zero;
                else
                    v[n1] = ok ? src[(int64_t)j * Nx + q] : zero;
            }
            reg_fft<R1, DIR>(v);
#pragma unroll
            for (int k1 = 1; k1 < R1; ++k1) {
                float2 w = __ldg(&tw[n2 * k1]);
                if (DIR > 0) w.y = -w.y;
                v[k1] = cmul(v[k1], w);
            }
#pragma unroll
            for (int k1 = 0; k1 < R1; ++k1) S[em_idx<N, Q>(n2 * R1 + k1, q)] = v[k1];
        }
        __syncthreads();
        if (threadIdx.x < R1 * Q) {
            const int k1 = threadIdx.x / Q, q = threadIdx.x % Q;
            if (kx0 + q >= Nx) return;
            float2 u[R2];
#pragma unroll
            for (int n2 = 0; n2 < R2; ++n2) u[n2] = S[em_idx<N, Q>(n2 * R1 + k1, q)];
            reg_fft<R2, DIR>(u);
#pragma unroll
            for (int k2 = 0; k2 < R2; ++k2) {
                const int j = k1 + R1 * k2;
                if (DIR < 0)
                    dst[(int64_t)j * Nx + q] = u[k2];
                else if (k2 < R2 / 2 && j < Lout && live(j))
                    dst[(int64_t)j * Nx + q] = u[k2];
            }
        }
    }
}

// cp.async helpers (16-byte LDGSTS, no register cost) for the staged strided pass
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }

// Staged strided pass (B / D) for 128 <= N <= 512.  X2 =
// [plane p = rc*Kz + z][ky < Ny][kx < Nx] is described by ONE 3-D tensor map (box 8 kx x
// 256 rows): the forward pass (B) stores its output tile with it, the inverse pass (D)
// loads its input tile with it, one cp.async.bulk.tensor per 256-row box into an
// mbarrier-tracked ring.  The other side keeps the pruned row traffic: B loads only the rows
// holding a voxel (cp.async, empty rows zero-filled in shared memory), D stores only those rows.
template <int N, int DIR, int S, int QQ>
struct YTma {
    static constexpr int Q = QQ;
    static constexpr int R1 = fft_r1(N), R2 = fft_r2(N);
    static constexpr int NT = R1 * Q;
    static constexpr int SR = DIR < 0 ? N / 2 : N;
    static constexpr int MW = (N / 2 + 31) / 32;
    static constexpr int BOX = N < 256 ? N : 256;
    static constexpr size_t stage_b = (size_t)SR * Q * sizeof(float2);
    static constexpr size_t T_b = ((size_t)em_size<N, Q>() * sizeof(float2) + 127) / 128 * 128;
    static constexpr size_t O_b = DIR < 0 ? (size_t)N * Q * sizeof(float2) : 0;
    static constexpr size_t smem = S * stage_b + T_b + O_b + (size_t)S * MW * 4 + S * 8 + 128;
};

template <int N, int DIR, int S, int QQ>
__global__ void __launch_bounds__(fft_r1(N) * QQ, (QQ == 4 && N <= 1024) ? 2 : 1)
    k_ytma(const float2* __restrict__ in, float2* __restrict__ out, const __grid_constant__ CUtensorMap tmap,
           const float2* __restrict__ tw, int Nx, int Kz, int Lin,
           int Lout, int ntiles, int tiles_x, const int32_t* __restrict__ planes, int nzp,
           const uint32_t* __restrict__ rowmask, int rowMW) {
    using P = YTma<N, DIR, S, QQ>;
    constexpr int Q = P::Q, R1 = P::R1, R2 = P::R2, NT = P::NT, SR = P::SR, MW = P::MW, BOX = P::BOX;
    constexpr int NL = DIR < 0 ? R1 / 2 : R1;
    constexpr bool TMA_IN = DIR > 0;
    constexpr int BOXI = SR < 256 ? SR : 256;
    extern __shared__ __align__(128) unsigned char smraw[];
    float2* stage = reinterpret_cast<float2*>(smraw);
    float2* T = reinterpret_cast<float2*>(smraw + S * P::stage_b);
    float2* O = reinterpret_cast<float2*>(smraw + S * P::stage_b + P::T_b);
    uint32_t* M = reinterpret_cast<uint32_t*>(smraw + S * P::stage_b + P::T_b + P::O_b);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smraw + ((S * P::stage_b + P::T_b + P::O_b + S * MW * 4 + 7) / 8) * 8);
    const int tid = threadIdx.x;
    const float2 zero = make_float2(0.f, 0.f);
    const int lin = min(Lin, SR);
    if (DIR < 0) {
        for (int e = tid; e < S * (SR - lin) * Q; e += NT) {
            const int st = e / ((SR - lin) * Q), r = e % ((SR - lin) * Q);
            stage[st * SR * Q + lin * Q + r] = zero;
        }
    } else if (tid == 0) {
        for (int st = 0; st < S; ++st) mbar_init(&bar[st], 1);
        mbar_fence_init();
    }
    __syncthreads();
    auto decode = [&](int t, int& z, int& p, int64_t& bin, int64_t& bout) {
        const int xt = t % tiles_x, pr = t / tiles_x;
        const int rc = pr / nzp;
        z = __ldg(&planes[pr - rc * nzp]);
        p = rc * Kz + z;
        bin = (int64_t)p * Lin * Nx + (int64_t)xt * Q;
        bout = (int64_t)p * Lout * Nx + (int64_t)xt * Q;
    };
    auto issue = [&](int t, int st) {
        if (!TMA_IN) {
            if (t < ntiles) {
                int z, p;
                int64_t bin, bout;
                decode(t, z, p, bin, bout);
                const uint32_t* pm = rowmask + (int64_t)z * rowMW;
                const float2* src = in + bin;
                float2* dst = stage + st * SR * Q;
                constexpr int NE = (SR * (Q / 2) + NT - 1) / NT;   // 16-byte chunks per thread
                uint32_t wd[NE];
#pragma unroll
                for (int k = 0; k < NE; ++k) {   // all mask words first: one load latency, not NE
                    const int j = (tid + k * NT) / (Q / 2);
                    wd[k] = j < lin ? __ldg(&pm[j >> 5]) : 0u;
                }
#pragma unroll
                for (int k = 0; k < NE; ++k) {
                    const int e = tid + k * NT;
                    const int j = e / (Q / 2), p2 = 2 * (e % (Q / 2));
                    if (j < lin) {
                        if ((wd[k] >> (j & 31)) & 1u)
                            cp_async16(dst + j * Q + p2, src + (int64_t)j * Nx + p2);
                        else
                            *reinterpret_cast<float4*>(dst + j * Q + p2) = make_float4(0.f, 0.f, 0.f, 0.f);
                    }
                }
            }
            cp_async_commit();
        } else if (t < ntiles) {
            int z, p;
            int64_t bin, bout;
            decode(t, z, p, bin, bout);
            if (tid < MW) M[st * MW + tid] = tid < rowMW ? __ldg(&rowmask[(int64_t)z * rowMW + tid]) : 0u;
            if (tid == 0) {
                mbar_arrive_expect_tx(&bar[st], (uint32_t)P::stage_b);
#pragma unroll
                for (int b = 0; b < SR / BOXI; ++b)
                    tma_load_3d(stage + st * SR * Q + b * BOXI * Q, &tmap, (t % tiles_x) * Q,
                                b * BOXI, p, &bar[st]);
            }
        }
    };
    const int n2 = tid / Q, q1 = tid % Q;
    const bool ph1 = n2 < R2;
    // phase-1 twiddles W_N^{n2 k1}: loop-invariant, in registers; for R1 = 64 (N = 2048) there is
    // no register room next to the 64-point transform, they are read from the (L1-resident) table
    constexpr bool TW_REG = R1 < 64;
    float2 tw1[TW_REG ? R1 : 1];
    if constexpr (TW_REG) {
#pragma unroll
        for (int kk = 1; kk < R1; ++kk) {
            float2 w = ph1 ? __ldg(&tw[n2 * kk]) : zero;
            if (DIR > 0) w.y = -w.y;
            tw1[kk] = w;
        }
    }
    const int k1 = tid / Q, q2 = tid % Q;
    int t = blockIdx.x;
#pragma unroll
    for (int s2 = 0; s2 < S - 1; ++s2) issue(t + s2 * (int)gridDim.x, s2);
    int pend_xt = 0, pend_p = -1;   // forward: output tile staged in O, store not yet issued
    for (int i = 0; t < ntiles; ++i, t += gridDim.x) {
        issue(t + (S - 1) * (int)gridDim.x, (i + S - 1) % S);
        const int st = i % S;
        if (!TMA_IN) {
            asm volatile("cp.async.wait_group %0;\n" ::"n"(S - 1));
        } else {
            mbar_wait(&bar[st], (uint32_t)((i / S) & 1));
        }
        __syncthreads();
        if (DIR < 0 && tid == 0 && pend_p >= 0) {
#pragma unroll
            for (int b = 0; b < N / BOX; ++b) tma_store_3d(&tmap, pend_xt, b * BOX, pend_p, O + b * BOX * Q);
            tma_store_commit();
        }
        int z, p;
        int64_t bin, bout;
        decode(t, z, p, bin, bout);
        if (ph1) {
            const float2* src = stage + st * SR * Q;
            float2 v[R1];
#pragma unroll
            for (int n1 = 0; n1 < R1; ++n1) {
                const int j = R2 * n1 + n2;
                v[n1] = n1 < NL ? src[j * Q + q1] : zero;
            }
            reg_fft<R1, DIR, (DIR < 0)>(v);
#pragma unroll
            for (int kk = 1; kk < R1; ++kk) {
                float2 w;
                if constexpr (TW_REG) {
                    w = tw1[kk];
                } else {
                    w = __ldg(&tw[n2 * kk]);
                    if (DIR > 0) w.y = -w.y;
                }
                v[kk] = cmul(v[kk], w);
            }
#pragma unroll
            for (int kk = 0; kk < R1; ++kk) T[em_idx<N, Q>(n2 * R1 + kk, q1)] = v[kk];
        }
        uint32_t keep = 0;
        if (DIR > 0) {
#pragma unroll
            for (int k2 = 0; k2 < R2 / 2; ++k2) {
                const int j = k1 + R1 * k2;
                if (j < Lout && ((M[st * MW + (j >> 5)] >> (j & 31)) & 1u)) keep |= 1u << k2;
            }
        }
        if (DIR < 0 && tid == 0) tma_store_wait_read0();   // O of the previous tile has been read out
        __syncthreads();
        float2 u[R2];
#pragma unroll
        for (int m = 0; m < R2; ++m) u[m] = T[em_idx<N, Q>(m * R1 + k1, q2)];
        reg_fft<R2, DIR>(u);
        if (DIR < 0) {
            // staged for the TMA store, which thread 0 issues after the NEXT tile's top barrier
            // (that barrier orders these writes; no extra barrier per tile)
#pragma unroll
            for (int k2 = 0; k2 < R2; ++k2) O[(k1 + R1 * k2) * Q + q2] = u[k2];
            fence_proxy_async_smem();
            pend_xt = (t % tiles_x) * Q;
            pend_p = p;
        } else {
            float2* dst = out + bout + q2;
#pragma unroll
            for (int k2 = 0; k2 < R2 / 2; ++k2)
                if ((keep >> k2) & 1u) dst[(k1 + R1 * k2) * Nx] = u[k2];
        }
    }
    if (DIR < 0) {
        asm volatile("cp.async.wait_group 0;\n" ::);
        __syncthreads();
        if (tid == 0) {
            if (pend_p >= 0) {
#pragma unroll
                for (int b = 0; b < N / BOX; ++b) tma_store_3d(&tmap, pend_xt, b * BOX, pend_p, O + b * BOX * Q);
                tma_store_commit();
            }
            tma_store_wait0();
        }
    }
}

// ---------------------------------------------------------------------------
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
    const float2 P1x = cfma_s(m1x, k2x, cmul_i(Ix, s1x));
    const float2 P1y = cfma_s(m1y, k2y, cmul_i(Iy, s1y));
    const float2 P1z = cfma_s(m1z, k2z, cmul_i(Iz, s1z));
    const float2 C2 = csub(P1x, P1y);
    const float2 C3 = cfma_s(P1z, -2.f, cadd(P1x, P1y));
    v[0] = cmul_i(P0x, g);
    v[1] = cmul_i(P0y, g);
    v[2] = cmul_i(P0z, g);
    v[3] = cmul_i(C2, g);
    v[4] = cmul_i(C3, g);
}


// Tucker expansion of the 7 kernel spectra for a CTA tile (fixed ky, Q consecutive kx, all N kz)
// into KV[m][kz][q]: G = core x2 F2[oy] (d3 x d1), H[q] = G x1 F1[ox_q] (d3), KV = H x3 F3[oz].
// scratch: >= 2 * 32 * max(Q, 32) floats of shared memory.
template <int N, int Q>
__device__ void tucker_tile(const SpecView& sv, int kx0, int ky, int Nx, int Ny, float* KV, float* scratch) {
    const int oy = ky <= (Ny >> 1) ? ky : Ny - ky;
    const float sy = ky <= (Ny >> 1) ? 1.f : -1.f;
    float* G = scratch;            // [d3][d1]
    float* H = scratch + 32 * 32;  // [Q][d3]
#pragma unroll
    for (int m = 0; m < 7; ++m) {
        const int d1 = sv.rk[m][0], d2 = sv.rk[m][1], d3 = sv.rk[m][2];
        const float* C = sv.core[m];
        const float* F1 = sv.fac[m][0];
        const float* F2 = sv.fac[m][1] + (int64_t)oy * d2;
        const float* F3 = sv.fac[m][2];
        for (int t = threadIdx.x; t < d3 * d1; t += blockDim.x) {
            const int c3 = t / d1, c1 = t % d1;
            float acc = 0.f;
            for (int c2 = 0; c2 < d2; ++c2) acc = fmaf(__ldg(&C[((int64_t)c3 * d2 + c2) * d1 + c1]), __ldg(&F2[c2]), acc);
            G[t] = acc;
        }
        __syncthreads();
        for (int t = threadIdx.x; t < Q * d3; t += blockDim.x) {
            const int q = t / d3, c3 = t % d3;
            const int kx = min(kx0 + q, Nx - 1);
            const int ox = kx <= (Nx >> 1) ? kx : Nx - kx;
            const float* f1 = F1 + (int64_t)ox * d1;
            float acc = 0.f;
            for (int c1 = 0; c1 < d1; ++c1) acc = fmaf(G[c3 * d1 + c1], __ldg(&f1[c1]), acc);
            H[t] = acc;
        }
        __syncthreads();
        for (int t = threadIdx.x; t < N * Q; t += blockDim.x) {
            const int k = t / Q, q = t % Q;
            const int kx = min(kx0 + q, Nx - 1);
            const int oz = k <= (N >> 1) ? k : N - k;
            const float* f3 = F3 + (int64_t)oz * d3;
            float acc = 0.f;
            for (int c3 = 0; c3 < d3; ++c3) acc = fmaf(H[q * d3 + c3], __ldg(&f3[c3]), acc);
            float sgn = 1.f;
            if (m == 1) sgn = kx <= (Nx >> 1) ? 1.f : -1.f;
            if (m == 2) sgn = sy;
            if (m == 3) sgn = k <= (N >> 1) ? 1.f : -1.f;
            KV[(m * N + k) * Q + q] = sgn * acc;
        }
        __syncthreads();
    }
}

// the 7 kernel spectra at frequency (kx, ky, kz) from the octant (mirror symmetry + parity)
__device__ __forceinline__ void kernel_values(const SpecView& sv, int kx, int ky, int kz, int Nx, int Ny, int Nz,
                                              float (&kv)[7]) {
    const int ox = kx <= (Nx >> 1) ? kx : Nx - kx;
    const int oy = ky <= (Ny >> 1) ? ky : Ny - ky;
    const int oz = kz <= (Nz >> 1) ? kz : Nz - kz;
    const float sx = kx <= (Nx >> 1) ? 1.f : -1.f;
    const float sy = ky <= (Ny >> 1) ? 1.f : -1.f;
    const float sz = kz <= (Nz >> 1) ? 1.f : -1.f;
    const int64_t pl = (int64_t)sv.hx * sv.hy * sv.hz;
    const int64_t o = ((int64_t)oz * sv.hy + oy) * sv.hx + ox;
#pragma unroll
    for (int k = 0; k < 7; ++k) kv[k] = __ldg(&sv.spec[k * pl + o]);
    kv[1] *= sx;
    kv[2] *= sy;
    kv[3] *= sz;
}

template <int N, int Q>
__host__ __device__ constexpr int freq_small_spec_f2() {
    return 5 * N * Q > (1024 + 32 * Q + 1) / 2 ? 5 * N * Q : (1024 + 32 * Q + 1) / 2;
}
template <int N, int Q, bool ASYNC>
constexpr size_t freq_small_smem() {
    return (size_t)freq_small_spec_f2<N, Q>() * sizeof(float2) + (size_t)7 * N * Q * sizeof(float) +
           (ASYNC ? (size_t)5 * ((N + 1) / 2) * Q * sizeof(float2) : 0);
}

// Pass C for Nz <= 64: one thread per (component, pencil) does the whole
// z-FFT in registers; the 5 spectra of Q pencils meet in shared memory for
// the MAC.  The CTA loops over all RHS of the batch (the 7 kernel spectra of
// its points are computed once into shared memory) and prefetches the next
// RHS while the current one is transformed: into registers (ASYNC = false) or
// into a shared staging tile with cp.async (ASYNC = true).
template <int N, int Q, bool ASYNC>
__global__ void __launch_bounds__(5 * Q)
    k_freq_small(float2* __restrict__ X2, SpecView sv, int Nx, int Ny, int Kz, float g, int nrhs, uint64_t pmask,
                 int Nxs, int kxg) {
    extern __shared__ float2 S[];   // [5][N][Q] spectra (also Tucker scratch), [7][N][Q] kernel values, stage
    float* KV = reinterpret_cast<float*>(S + freq_small_spec_f2<N, Q>());
    constexpr int NH = (N + 1) / 2;
    float2* stage = reinterpret_cast<float2*>(KV + 7 * N * Q);   // [5][NH][Q]
    const int c = threadIdx.x / Q, q = threadIdx.x % Q;
    const int kx0 = blockIdx.x * Q;
    const int ky = blockIdx.y;
    const int64_t plane = (int64_t)Nxs * Ny;   // array x-extent (a kx-slab: Nx/P)
    const bool ok = kx0 + q < Nxs;
    const float2 zero = make_float2(0.f, 0.f);
    float2* col = X2 + (int64_t)c * Kz * plane + (int64_t)ky * Nxs + kx0 + q;
    const int64_t rstride = 5 * Kz * plane;
    const int kz_ld = min(Kz, NH);
    auto issue = [&](int r) {   // cp.async the RHS r tile: 5 comps x kz_ld rows x Q columns (16-byte chunks)
        const float2* base = X2 + r * rstride + (int64_t)ky * Nxs + kx0;
        for (int e = threadIdx.x; e < 5 * kz_ld * (Q / 2); e += 5 * Q) {
            const int p = e % (Q / 2), rest = e / (Q / 2);
            const int j = rest % kz_ld, cc = rest / kz_ld;
            if ((pmask >> j) & 1u)
                cp_async16(stage + (cc * NH + j) * Q + 2 * p, base + ((int64_t)cc * Kz + j) * plane + 2 * p);
        }
    };
    float2 nxt[ASYNC ? 1 : NH];
    if constexpr (ASYNC) {
        issue(0);
        cp_async_commit();
    } else {
#pragma unroll
        for (int j = 0; j < NH; ++j) nxt[j] = (ok && j < Kz && ((pmask >> j) & 1u)) ? col[(int64_t)j * plane] : zero;
    }
    // the 7 kernel spectra of this CTA's (kz, kx) points, reused by every RHS:
    // dense octant lookup, or Tucker expansion on chip (scratch = the spectra buffer)
    if (sv.spec) {
        for (int t = threadIdx.x; t < N * Q; t += 5 * Q) {
            const int k = t / Q, qq = t % Q;
            float kv[7];
            kernel_values(sv, min(kxg + kx0 + qq, Nx - 1), ky, k, Nx, Ny, N, kv);
#pragma unroll
            for (int m = 0; m < 7; ++m) KV[(m * N + k) * Q + qq] = kv[m];
        }
    } else {
        tucker_tile<N, Q>(sv, kxg + kx0, ky, Nx, Ny, KV, reinterpret_cast<float*>(S));
    }
    for (int r = 0; r < nrhs; ++r) {
        float2 v[N];
        if constexpr (ASYNC) {
            asm volatile("cp.async.wait_group 0;\n" ::);
            __syncthreads();
#pragma unroll
            for (int j = 0; j < N; ++j) v[j] = (j < NH && j < Kz && ((pmask >> j) & 1u)) ? stage[(c * NH + j) * Q + q] : zero;
            __syncthreads();
            if (r + 1 < nrhs) issue(r + 1);
            cp_async_commit();
        } else {
#pragma unroll
            for (int j = 0; j < N; ++j) v[j] = j < NH ? nxt[j] : zero;
        }
        reg_fft<N, -1>(v);
#pragma unroll
        for (int k = 0; k < N; ++k) S[(c * N + k) * Q + q] = v[k];
        __syncthreads();
        if constexpr (!ASYNC) {
            if (r + 1 < nrhs) {
                const float2* nc = col + (r + 1) * rstride;
#pragma unroll
                for (int j = 0; j < NH; ++j) nxt[j] = (ok && j < Kz && ((pmask >> j) & 1u)) ? nc[(int64_t)j * plane] : zero;
            }
        }
        for (int t = threadIdx.x; t < N * Q; t += 5 * Q) {
            const int k = t / Q, qq = t % Q;
            float2 w[5];
#pragma unroll
            for (int cc = 0; cc < 5; ++cc) w[cc] = S[(cc * N + k) * Q + qq];
            mac5(w, KV[(0 * N + k) * Q + qq], KV[(1 * N + k) * Q + qq], KV[(2 * N + k) * Q + qq],
                 KV[(3 * N + k) * Q + qq], KV[(4 * N + k) * Q + qq], KV[(5 * N + k) * Q + qq],
                 KV[(6 * N + k) * Q + qq], g);
#pragma unroll
            for (int cc = 0; cc < 5; ++cc) S[(cc * N + k) * Q + qq] = w[cc];
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < N; ++k) v[k] = S[(c * N + k) * Q + q];
        reg_fft<N, +1>(v);
        if (ok) {
            float2* dst = col + r * rstride;
#pragma unroll
            for (int j = 0; j < NH; ++j)
                if (j < Kz && ((pmask >> j) & 1u)) dst[(int64_t)j * plane] = v[j];
        }
    }
}

// Pass C, default for 2 <= Nz <= 32: 32 pencils (kx) x 5 components per CTA, one
// thread per (component, pencil) for the z-FFTs in registers, the CTA loops over all
// RHS (register prefetch of the next one):
//  * the prefactor j*omega*mu0*dx/(Nx Ny Nz) and the constants of the moment form are
//    folded into the 7 kernel values once per CTA, so the MAC is 19 paired-FP32 ops;
//  * the MAC points are split warp-uniformly (warp w takes kz = w, w+5, ...; lane = kx),
//    all shared-memory offsets are compile-time;
//  * the forward z-FFT skips its zero-padded half (reg_fft HALF_IN).
// Folded values per point (K1 = -i s1):
//   f0 = g K0, f1 = g s1x, f2 = g s1y, f3 = -2 g s1z, f4 = g K2x, f5 = g K2y, f6 = 4 g K2z
//   CCx = i f0 Ix + f1 m1x,  CCy = i f0 Iy + f2 m1y,  CCz = i f0 Iz + f3 I3
//   Qx = -f1 Ix + i f4 m1x,  Qy = -f2 Iy + i f5 m1y,  Qz' = -2 Qz = -f3 Iz + i f6 I3
//   CC2D = Qx - Qy,  CC3D = Qx + Qy + Qz'          (m1x = I2D + I3D, m1y = I3D - I2D)
template <int N>
constexpr int zmac_s_f2() {   // spectra buffer, also >= the 2048-float Tucker scratch
    return 5 * N * 32 > 1024 ? 5 * N * 32 : 1024;
}
template <int N>
constexpr size_t zmac_smem() {
    return (size_t)zmac_s_f2<N>() * sizeof(float2) + (size_t)7 * N * 32 * sizeof(float);
}

template <int N>
__global__ void __launch_bounds__(160, 3)
    k_zmac(float2* __restrict__ X2, SpecView sv, int Nx, int Ny, int Kz, float g, int nrhs, uint64_t pmask, int Nxs,
           int kxg, int zpre) {
    constexpr int Q = 32, NH = N / 2;
    extern __shared__ float2 S[];                       // [5][N][Q] spectra; Tucker scratch
    float* KV = reinterpret_cast<float*>(S + zmac_s_f2<N>());   // [7][N][Q] folded kernel values
    const int tid = threadIdx.x;
    const int c = tid >> 5, q = tid & 31;               // FFT role: component c, pencil q
    const int kx0 = blockIdx.x * Q;
    const int ky = blockIdx.y;
    const int64_t plane = (int64_t)Nxs * Ny;   // array x-extent (a kx-slab: Nx/P)
    const bool ok = kx0 + q < Nxs;
    const float2 zero = make_float2(0.f, 0.f);
    float2* col = X2 + (int64_t)c * Kz * plane + (int64_t)ky * Nxs + kx0 + q;
    const int64_t rstride = 5 * Kz * plane;
    // rows z < min(Kz, N/2) of non-empty planes are loaded / stored; the rest are zero / dropped
    const uint32_t lm = ok ? (uint32_t)(pmask & ((1ull << min(Kz, NH)) - 1ull)) : 0u;
    float2 nxt[NH];
#pragma unroll
    for (int j = 0; j < NH; ++j) nxt[j] = ((lm >> j) & 1u) ? col[(int64_t)j * plane] : zero;
    const float fold[7] = {g, g, g, -2.f * g, g, g, 4.f * g};
    if (sv.spec) {
        // dense octant lookup, folded: warp c takes kz = c + 5 i, lane = kx (coalesced along
        // the octant's x rows); all 7 x ceil(N/5) loads are independent and issued together
        const int kx = min(kxg + kx0 + q, Nx - 1);
        const int ox = kx <= (Nx >> 1) ? kx : Nx - kx;
        const int oy = ky <= (Ny >> 1) ? ky : Ny - ky;
        const float sx = kx <= (Nx >> 1) ? 1.f : -1.f, sy = ky <= (Ny >> 1) ? 1.f : -1.f;
        const int64_t pl = (int64_t)sv.hx * sv.hy * sv.hz;
        float kv[(N + 4) / 5][7];
#pragma unroll
        for (int i = 0; i < (N + 4) / 5; ++i) {
            const int k = c + 5 * i;
            const int oz = (k < N ? (k <= (N >> 1) ? k : N - k) : 0);
            const int64_t o = ((int64_t)oz * sv.hy + oy) * sv.hx + ox;
#pragma unroll
            for (int m = 0; m < 7; ++m) kv[i][m] = __ldg(&sv.spec[m * pl + o]);
        }
#pragma unroll
        for (int i = 0; i < (N + 4) / 5; ++i) {
            const int k = c + 5 * i;
            if (k < N) {
                const float sz = k <= (N >> 1) ? 1.f : -1.f;
                const float sgn[7] = {1.f, sx, sy, sz, 1.f, 1.f, 1.f};
#pragma unroll
                for (int m = 0; m < 7; ++m) KV[(m * N + k) * Q + q] = kv[i][m] * sgn[m] * fold[m];
            }
        }
    } else {
        tucker_tile<N, Q>(sv, kxg + kx0, ky, Nx, Ny, KV, reinterpret_cast<float*>(S));
        __syncthreads();
        for (int t = tid; t < 7 * N * Q; t += 5 * Q) {
            const int m = t / (N * Q);
            KV[t] *= m == 3 ? -2.f * g : (m == 6 ? 4.f * g : g);
        }
    }
    // MAC role: warp w = c takes kz = w + 5 i; lane = pencil
    const int w = c;
    for (int r = 0; r < nrhs; ++r) {
        float2 v[N];
#pragma unroll
        for (int j = 0; j < N; ++j) v[j] = j < NH ? nxt[j] : zero;
        reg_fft<N, -1, true>(v);
#pragma unroll
        for (int k = 0; k < N; ++k) S[(c * N + k) * Q + q] = v[k];
        __syncthreads();
        if (r + 1 < nrhs) {
            const float2* nc = col + (r + 1) * rstride;
#pragma unroll
            for (int j = 0; j < NH; ++j) nxt[j] = ((lm >> j) & 1u) ? nc[(int64_t)j * plane] : zero;
        }
        // the RHS after next: its rows of this tile are bulk-prefetched into L2 (one
        // 256-byte cp.async.bulk.prefetch per (component, z) row, no registers), so the
        // register prefetch above hits L2 one iteration later
        if (zpre && r + 2 < nrhs && tid < 5 * NH) {
            const int cc = tid / NH, j = tid % NH;
            const int nb = min(Q, Nxs - kx0) * 8 / 16 * 16;
            if (j < Kz && ((pmask >> j) & 1u) && nb > 0) {
                const float2* a = X2 + (r + 2) * rstride + ((int64_t)cc * Kz + j) * plane + (int64_t)ky * Nxs + kx0;
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(a), "r"(nb) : "memory");
            }
        }
        float2* sp = S + w * Q + q;
        const float* kp = KV + w * Q + q;
#pragma unroll 1
        for (int k = w; k < N ; k += 5, sp += 5 * Q, kp += 5 * Q) {
            {
                const float2 Ix = sp[0 * N * Q], Iy = sp[1 * N * Q], Iz = sp[2 * N * Q];
                const float2 I2 = sp[3 * N * Q], I3 = sp[4 * N * Q];
                const float f0 = kp[0 * N * Q], f1 = kp[1 * N * Q], f2 = kp[2 * N * Q], f3 = kp[3 * N * Q];
                const float f4 = kp[4 * N * Q], f5 = kp[5 * N * Q], f6 = kp[6 * N * Q];
                const float2 m1x = cadd(I2, I3), m1y = csub(I3, I2);
                const float2 Qx = cfma_s(Ix, -f1, cmul_i(m1x, f4));
                const float2 Qy = cfma_s(Iy, -f2, cmul_i(m1y, f5));
                const float2 Qz = cfma_s(Iz, -f3, cmul_i(I3, f6));
                sp[0 * N * Q] = cfma_s(m1x, f1, cmul_i(Ix, f0));
                sp[1 * N * Q] = cfma_s(m1y, f2, cmul_i(Iy, f0));
                sp[2 * N * Q] = cfma_s(I3, f3, cmul_i(Iz, f0));
                sp[3 * N * Q] = csub(Qx, Qy);
                sp[4 * N * Q] = cadd(cadd(Qx, Qy), Qz);
            }
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < N; ++k) v[k] = S[(c * N + k) * Q + q];   // own column: no barrier before reuse
        reg_fft<N, +1>(v);
        float2* dst = col + r * rstride;
#pragma unroll
        for (int j = 0; j < NH; ++j)
            if ((lm >> j) & 1u) dst[(int64_t)j * plane] = v[j];
    }
}

// Pass C, occupancy variant (dense octant spectra, Nz <= 32): the kernel values are kept for
// kz <= Nz/2 only (K0, K1x, K1y, K2 are even in kz, K1z odd: 15 KB instead of 28 KB) and the
// next RHS is not staged in registers but bulk-prefetched into L2 (cp.async.bulk.prefetch), so
// a CTA needs <= 96 registers / thread and ~55 KB of shared memory: 4 CTAs (20 warps) per SM
// instead of 3.  Same arithmetic as k_zmac.
template <int N>
constexpr size_t zmac2_smem() {
    return (size_t)zmac_s_f2<N>() * sizeof(float2) + (size_t)7 * (N / 2 + 1) * 32 * sizeof(float);
}

template <int N>
__global__ void __launch_bounds__(160, 4)
    k_zmac2(float2* __restrict__ X2, SpecView sv, int Nx, int Ny, int Kz, float g, int nrhs, uint64_t pmask, int Nxs,
            int kxg) {
    constexpr int Q = 32, NH = N / 2, NK = N / 2 + 1;
    constexpr int NS = N;                                // kz rows held in S
    extern __shared__ float2 S[];
    float* KV = reinterpret_cast<float*>(S + zmac_s_f2<N>());   // [7][NK][Q]
    const int tid = threadIdx.x;
    const int c = tid >> 5, q = tid & 31;
    const int kx0 = blockIdx.x * Q;
    const int ky = blockIdx.y;
    const int64_t plane = (int64_t)Nxs * Ny;
    const bool ok = kx0 + q < Nxs;
    const float2 zero = make_float2(0.f, 0.f);
    float2* col = X2 + (int64_t)c * Kz * plane + (int64_t)ky * Nxs + kx0 + q;
    const int64_t rstride = 5 * Kz * plane;
    const uint32_t lm = ok ? (uint32_t)(pmask & ((1ull << min(Kz, NH)) - 1ull)) : 0u;
    const int nb = min(Q, Nxs - kx0) * 8 / 16 * 16;
    auto prefetch = [&](int r) {   // this tile's rows of RHS r -> L2
        if (r < nrhs && tid < 5 * NH) {
            const int cc = tid / NH, j = tid % NH;
            if (j < Kz && ((pmask >> j) & 1u) && nb > 0) {
                const float2* a = X2 + r * rstride + ((int64_t)cc * Kz + j) * plane + (int64_t)ky * Nxs + kx0;
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(a), "r"(nb) : "memory");
            }
        }
    };
    prefetch(0);
    prefetch(1);
    {
        const int kx = min(kxg + kx0 + q, Nx - 1);
        const int ox = kx <= (Nx >> 1) ? kx : Nx - kx;
        const int oy = ky <= (Ny >> 1) ? ky : Ny - ky;
        const float sx = kx <= (Nx >> 1) ? 1.f : -1.f, sy = ky <= (Ny >> 1) ? 1.f : -1.f;
        const float fold[7] = {g, g * sx, g * sy, -2.f * g, g, g, 4.f * g};
        const int64_t pl = (int64_t)sv.hx * sv.hy * sv.hz;
#pragma unroll
        for (int i = 0; i < (NK + 4) / 5; ++i) {
            const int k = c + 5 * i;
            if (k < NK) {
                const int64_t o = ((int64_t)k * sv.hy + oy) * sv.hx + ox;
#pragma unroll
                for (int m = 0; m < 7; ++m) KV[(m * NK + k) * Q + q] = __ldg(&sv.spec[m * pl + o]) * fold[m];
            }
        }
    }
    const int w = c;
    for (int r = 0; r < nrhs; ++r) {
        float2 v[N];
        const float2* src = col + r * rstride;
#pragma unroll
        for (int j = 0; j < N; ++j) v[j] = (j < NH && ((lm >> j) & 1u)) ? src[(int64_t)j * plane] : zero;
        prefetch(r + 2);
        reg_fft<N, -1, true>(v);
#pragma unroll
        for (int hh = 0; hh < 1; ++hh) {
            const int k0 = hh * NS;   // kz rows [k0, k0 + NS) in S
#pragma unroll
            for (int k = 0; k < NS; ++k) S[(c * NS + k) * Q + q] = v[k0 + k];
            __syncthreads();
#pragma unroll 1
            for (int kk = w; kk < NS; kk += 5) {
                const int k = k0 + kk;
                const int kh = k <= NH ? k : N - k;
                const float s3 = k <= NH ? 1.f : -1.f;   // K1z is odd in kz
                float2* sp = S + kk * Q + q;
                const float* kp = KV + kh * Q + q;
                const float2 Ix = sp[0 * NS * Q], Iy = sp[1 * NS * Q], Iz = sp[2 * NS * Q];
                const float2 I2 = sp[3 * NS * Q], I3 = sp[4 * NS * Q];
                const float f0 = kp[0 * NK * Q], f1 = kp[1 * NK * Q], f2 = kp[2 * NK * Q], f3 = s3 * kp[3 * NK * Q];
                const float f4 = kp[4 * NK * Q], f5 = kp[5 * NK * Q], f6 = kp[6 * NK * Q];
                const float2 m1x = cadd(I2, I3), m1y = csub(I3, I2);
                const float2 Qx = cfma_s(Ix, -f1, cmul_i(m1x, f4));
                const float2 Qy = cfma_s(Iy, -f2, cmul_i(m1y, f5));
                const float2 Qz = cfma_s(Iz, -f3, cmul_i(I3, f6));
                sp[0 * NS * Q] = cfma_s(m1x, f1, cmul_i(Ix, f0));
                sp[1 * NS * Q] = cfma_s(m1y, f2, cmul_i(Iy, f0));
                sp[2 * NS * Q] = cfma_s(I3, f3, cmul_i(Iz, f0));
                sp[3 * NS * Q] = csub(Qx, Qy);
                sp[4 * NS * Q] = cadd(cadd(Qx, Qy), Qz);
            }
            __syncthreads();
#pragma unroll
            for (int k = 0; k < NS; ++k) v[k0 + k] = S[(c * NS + k) * Q + q];   // own column
        }
        reg_fft<N, +1>(v);
        float2* dst = col + r * rstride;
#pragma unroll
        for (int j = 0; j < NH; ++j)
            if ((lm >> j) & 1u) dst[(int64_t)j * plane] = v[j];
    }
}

// Pass C for Nz > 64: generic shared-memory FFT over 5Q pencils (smem_fft).
// CTA size: smem_fft needs >= 5 Q x max(R1, R2) threads; with Q = 1 and R1 = 64 (N >= 2048)
// that is 320, above fft_max_threads(N)
template <int N>
constexpr int freq_big_threads() {
    return fft_max_threads(N) > 5 * fft_threads_per_pencil(N) ? fft_max_threads(N) : 5 * fft_threads_per_pencil(N);
}

template <int N>
__global__ void __launch_bounds__(freq_big_threads<N>())
    k_freq_big(float2* __restrict__ X2, SpecView sv, const float2* __restrict__ tw, int Nx, int Ny, int Kz, int Q,
               float g, const uint8_t* __restrict__ planeok, int Nxs, int kxg) {
    extern __shared__ float2 S[];
    const int Q5 = 5 * Q;
    const int PP = Q5 + 1;
    const int kx0 = blockIdx.x * Q;
    const int ky = blockIdx.y;
    const int64_t r = blockIdx.z;
    const int64_t plane = (int64_t)Nxs * Ny;
    float2* base = X2 + r * 5 * Kz * plane + (int64_t)ky * Nxs + kx0;
    const int nq = min(Q, Nxs - kx0);
    for (int t = threadIdx.x; t < Q * N * 5; t += blockDim.x) {
        const int q = t % Q;
        const int rest = t / Q;
        const int j = rest % N, c = rest / N;
        float2 v = make_float2(0.f, 0.f);
        if (j < Kz && q < nq && __ldg(&planeok[j])) v = base[((int64_t)c * Kz + j) * plane + q];
        S[j * PP + c * Q + q] = v;
    }
    // Tucker mode (Eq. 10): separable on-chip expansion, as tucker_tile: per CTA
    // G_m = core_m x2 F2[oy] (d3 x d1), H_m[q] = G_m x1 F1[ox_q] (d3); per point one d3-term
    // dot product with the F3 row of its kz (the dense circulant never exists in HBM)
    __shared__ float Gs[32 * 32];
    __shared__ float Hs[7][8][32];
    if (!sv.spec) {
        const int oy = ky <= (Ny >> 1) ? ky : Ny - ky;
        for (int m = 0; m < 7; ++m) {
            const int d1 = sv.rk[m][0], d2 = sv.rk[m][1], d3 = sv.rk[m][2];
            const float* C = sv.core[m];
            const float* F2 = sv.fac[m][1] + (int64_t)oy * d2;
            for (int t = threadIdx.x; t < d3 * d1; t += blockDim.x) {
                const int c3 = t / d1, c1 = t % d1;
                float acc = 0.f;
                for (int c2 = 0; c2 < d2; ++c2) acc = fmaf(__ldg(&C[((int64_t)c3 * d2 + c2) * d1 + c1]), __ldg(&F2[c2]), acc);
                Gs[t] = acc;
            }
            __syncthreads();
            for (int t = threadIdx.x; t < Q * d3; t += blockDim.x) {
                const int q = t / d3, c3 = t % d3;
                const int kx = min(kxg + kx0 + q, Nx - 1);
                const int ox = kx <= (Nx >> 1) ? kx : Nx - kx;
                const float* f1 = sv.fac[m][0] + (int64_t)ox * d1;
                float acc = 0.f;
                for (int c1 = 0; c1 < d1; ++c1) acc = fmaf(Gs[c3 * d1 + c1], __ldg(&f1[c1]), acc);
                Hs[m][q][c3] = acc;
            }
            __syncthreads();
        }
    }
    __syncthreads();
    smem_fft<N, -1>(S, PP, Q5, tw);
    for (int t = threadIdx.x; t < Q * N; t += blockDim.x) {
        const int q = t % Q, kz = t / Q;
        if (q >= nq) continue;
        float kv[7];
        if (sv.spec) {
            kernel_values(sv, kxg + kx0 + q, ky, kz, Nx, Ny, N, kv);
        } else {
            const int kx = kxg + kx0 + q;
            const int oz = kz <= (N >> 1) ? kz : N - kz;
#pragma unroll
            for (int m = 0; m < 7; ++m) {
                const int d3 = sv.rk[m][2];
                const float* f3 = sv.fac[m][2] + (int64_t)oz * d3;
                float acc = 0.f;
                for (int c3 = 0; c3 < d3; ++c3) acc = fmaf(Hs[m][q][c3], __ldg(&f3[c3]), acc);
                kv[m] = acc;
            }
            kv[1] *= kx <= (Nx >> 1) ? 1.f : -1.f;
            kv[2] *= ky <= (Ny >> 1) ? 1.f : -1.f;
            kv[3] *= kz <= (N >> 1) ? 1.f : -1.f;
        }
        float2 v[5];
#pragma unroll
        for (int c = 0; c < 5; ++c) v[c] = S[kz * PP + c * Q + q];
        mac5(v, kv[0], kv[1], kv[2], kv[3], kv[4], kv[5], kv[6], g);
#pragma unroll
        for (int c = 0; c < 5; ++c) S[kz * PP + c * Q + q] = v[c];
    }
    __syncthreads();
    smem_fft<N, +1>(S, PP, Q5, tw);
    for (int t = threadIdx.x; t < Q * Kz * 5; t += blockDim.x) {
        const int q = t % Q;
        const int rest = t / Q;
        const int j = rest % Kz, c = rest / Kz;
        if (q < nq && __ldg(&planeok[j])) base[((int64_t)c * Kz + j) * plane + q] = S[j * PP + c * Q + q];
    }
}

// Pass C for 128 <= Nz <= 512 (TMA-staged): a persistent CTA per SM walks tiles of one RHS x
// Q consecutive kx x one ky.  The tile's 5 x Kz x Q input block arrives by five
// cp.async.bulk.tensor loads (box Q x 1 x Kz, one per component) into a double-buffered
// mbarrier ring, so the load of the next tile overlaps this tile's transforms; the result
// leaves the same way (five TMA stores from the consumed input slot).  The z-FFT is the
// two-level R1 x R2 register/shared-memory transform of the strided passes (first level
// pruned to the Kz <= N/2 live inputs), the 5 spectra meet in shared memory in natural kz
// order for the moment-form MAC (mac5), and the inverse runs the transposed two-level
// transform, cropped to z < Kz.  Rows of planes without voxels are read as zero (X2 there is
// never written by pass B); their results are written but never read (pass D skips them).
// Pass C for Nz = 512 (k_zpass covers 64..256): tiles of one RHS x Q kx x one ky arrive by
// five cp.async.bulk.tensor loads (box Q x 1 x Kz) into a 2-slot mbarrier ring and leave by
// five TMA stores.  The z-FFT is split N = R1 x R2 with a SHORT second level (R2 = 8) so that one
// thread holds all 5 components of its (k1, q) column after the forward second level: the
// moment-form MAC then runs in registers (no spectrum round trip through shared memory),
// followed directly by the inverse first level, written back over the very elements the
// thread read (no barrier).  Per tile: 2 shared-memory transposes instead of 4 plus the MAC
// exchange.  The 7 kernel spectra of a (kx tile, ky) column are folded into shared memory
// once per group of nrhs tiles (the CTA walks all RHS of a column back to back).
template <int N, int Q, int R2_>
struct ZTma2 {
    static constexpr int R2 = R2_, R1 = N / R2_, NH = N / 2, NK = N / 2 + 1;
    static constexpr int NT1 = 5 * R2 * Q, NT2 = R1 * Q, NT = NT1 > NT2 ? NT1 : NT2;
    static constexpr int PADQ = Q < 16 ? Q : 0;
    static constexpr int EM = N * Q + R2 * PADQ;   // per component
    static constexpr int SLOT = 5 * NH * Q;
    static constexpr size_t stage_b = (size_t)SLOT * sizeof(float2);
    static constexpr size_t T_b = ((size_t)5 * EM * sizeof(float2) + 127) / 128 * 128;
    static constexpr size_t KV_b = ((size_t)7 * NK * Q * sizeof(float) + 127) / 128 * 128;
    static constexpr size_t smem = 2 * stage_b + T_b + 2 * KV_b + (size_t)N * sizeof(float2) + NH + 16 + 128;
    static_assert(KV_b >= (32 * 32 + 32 * Q) * sizeof(float), "Tucker scratch must fit one KV buffer");
    // transpose-buffer index of element (n2, k1) of pencil q (padded per n2 block)
    static __device__ __forceinline__ int ti(int n2, int k1, int q) { return (n2 * R1 + k1) * Q + q + n2 * PADQ; }
};

template <int N, int Q, int R2_>
__global__ void __launch_bounds__(ZTma2<N, Q, R2_>::NT, (N <= 128 || (N < 512 && Q == 4)) ? 2 : 1)
    k_ztma2(const __grid_constant__ CUtensorMap tmap, SpecView sv, const float2* __restrict__ tw, int Nx, int Ny,
            int Kz, float g, int nrhs, int ngroups, int tiles_x, const uint8_t* __restrict__ planeok, int kxg) {
    using P = ZTma2<N, Q, R2_>;
    constexpr int R1 = P::R1, R2 = P::R2, NH = P::NH, NK = P::NK, NT = P::NT, NT1 = P::NT1, NT2 = P::NT2;
    constexpr int EM = P::EM, SLOT = P::SLOT;
    extern __shared__ __align__(128) unsigned char smraw[];
    float2* stage = reinterpret_cast<float2*>(smraw);                                  // [2][5][NH][Q]
    float2* T = reinterpret_cast<float2*>(smraw + 2 * P::stage_b);                     // [5][EM]
    float* KV0 = reinterpret_cast<float*>(smraw + 2 * P::stage_b + P::T_b);            // [2][7][NK][Q]
    float2* tws = reinterpret_cast<float2*>(smraw + 2 * P::stage_b + P::T_b + 2 * P::KV_b);
    uint8_t* pok = reinterpret_cast<uint8_t*>(tws + N);
    uint64_t* bar = reinterpret_cast<uint64_t*>(
        smraw + ((2 * P::stage_b + P::T_b + 2 * P::KV_b + N * sizeof(float2) + NH + 7) / 8) * 8);
    const int tid = threadIdx.x;
    const float2 zero = make_float2(0.f, 0.f);
    for (int j = tid; j < N; j += NT) tws[j] = __ldg(&tw[j]);
    for (int j = tid; j < NH; j += NT) pok[j] = (j < Kz && __ldg(&planeok[j])) ? 1 : 0;
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
    }
    __syncthreads();
    // this CTA's tile sequence: column groups blockIdx.x, +gridDim.x, ...; all RHS of a group
    auto group_of = [&](int s) { return (int)blockIdx.x + (s / nrhs) * (int)gridDim.x; };
    // group -> (kx tile, ky), ordered so that the mirror images of a column (kx -> Nx - kx,
    // ky -> Ny - ky), which read the same octant rows of the kernel spectra, are consecutive
    // groups (run at the same time on neighbouring CTAs): those rows are fetched from HBM once
    // and are L2 hits for the other three.  First the mirror quadruples {xs, tiles_x-1-xs} x
    // {j, Ny-j} (j = 1 .. Ny/2-1), then the self-mirrored rows ky = 0 and Ny/2.
    const int npair = (tiles_x >= 2 && Ny >= 4) ? ((Ny >> 1) - 1) * 2 * tiles_x : 0;
    auto column = [&](int grp, int& xt, int& ky) {
        if (grp < npair) {
            const int ysl = grp / (2 * tiles_x), rem = grp % (2 * tiles_x);
            const int xs = rem >> 2;
            xt = (rem & 1) ? tiles_x - 1 - xs : xs;
            ky = ((rem >> 1) & 1) ? Ny - (ysl + 1) : ysl + 1;
            return;
        }
        const int g2 = grp - npair;
        const int xi = g2 % tiles_x, yi = g2 / tiles_x;
        xt = (xi & 1) ? tiles_x - 1 - (xi >> 1) : (xi >> 1);
        if (npair > 0)
            ky = yi ? (Ny >> 1) : 0;
        else
            ky = yi == 0 ? 0 : yi == 1 ? (Ny >> 1) : ((yi & 1) ? Ny - (yi >> 1) : (yi >> 1));
    };
    auto issue = [&](int s, int st) {
        const int grp = group_of(s), r = s % nrhs;
        if (grp >= ngroups) return;
        int xt, ky;
        column(grp, xt, ky);
        mbar_arrive_expect_tx(&bar[st], (uint32_t)(5 * Kz * Q * sizeof(float2)));
#pragma unroll
        for (int c = 0; c < 5; ++c)
            tma_load_3d(stage + st * SLOT + c * NH * Q, &tmap, xt * Q, ky, (r * 5 + c) * Kz, &bar[st]);
    };
    const int c1 = tid / (R2 * Q), n2 = (tid / Q) % R2, q1 = tid % Q;   // level-1 roles
    const int k1 = tid / Q, q2 = tid % Q;                               // level-2 roles
    // the 7 kernel spectra of a column group (raw octant values; the folding factors are
    // applied in the MAC), fetched by cp.async one group ahead into a double buffer
    const bool tucker = sv.spec == nullptr;
    auto fetch_kv = [&](int gi) {
        const int grp = (int)blockIdx.x + gi * (int)gridDim.x;
        if (!tucker && grp < ngroups) {
            int xt, ky;
        column(grp, xt, ky);
            const int oy = ky <= (Ny >> 1) ? ky : Ny - ky;
            const int64_t pl = (int64_t)sv.hx * sv.hy * sv.hz;
            float* dst = KV0 + (gi & 1) * (P::KV_b / sizeof(float));
            for (int e = tid; e < 7 * NK * Q; e += NT) {
                const int q = e % Q, rest = e / Q;
                const int kh = rest % NK, m = rest / NK;
                const int kx = min(kxg + xt * Q + q, Nx - 1);
                const int ox = kx <= (Nx >> 1) ? kx : Nx - kx;
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(dst + e)),
                             "l"(sv.spec + m * pl + ((int64_t)kh * sv.hy + oy) * sv.hx + ox)
                             : "memory");
            }
        }
        cp_async_commit();
    };
    fetch_kv(0);
    if (tid == 0) issue(0, 0);
    for (int s = 0;; ++s) {
        const int grp = group_of(s), r = s % nrhs;
        if (grp >= ngroups) break;
        int xt, ky;
        column(grp, xt, ky);
        const int st = s & 1;
        float2* slot = stage + st * SLOT;
        if (r == 0) {   // next group's spectra; this group's (fetched one group ago) must have landed
            fetch_kv(s / nrhs + 1);
            cp_async_wait1();   // published by the barrier after level 1
            if (tucker) {
                // Tucker mode (Eq. 10): the column's octant rows from the factors, on
                // chip: G_m = core_m x2 F2[oy] (d3 x d1), H_m[q] = G_m x1 F1[ox_q] (d3), row kh =
                // H_m[q] . F3[kh] -- into buffer 0, buffer 1 is the scratch
                float* G = KV0 + P::KV_b / sizeof(float);
                float* H = G + 32 * 32;
                const int oy = ky <= (Ny >> 1) ? ky : Ny - ky;
                for (int m = 0; m < 7; ++m) {
                    const int d1 = sv.rk[m][0], d2 = sv.rk[m][1], d3 = sv.rk[m][2];
                    const float* C = sv.core[m];
                    const float* F2 = sv.fac[m][1] + (int64_t)oy * d2;
                    for (int t = tid; t < d3 * d1; t += NT) {
                        const int c3 = t / d1, cc1 = t % d1;
                        float acc = 0.f;
                        for (int cc2 = 0; cc2 < d2; ++cc2)
                            acc = fmaf(__ldg(&C[((int64_t)c3 * d2 + cc2) * d1 + cc1]), __ldg(&F2[cc2]), acc);
                        G[t] = acc;
                    }
                    __syncthreads();
                    for (int t = tid; t < Q * d3; t += NT) {
                        const int q = t / d3, c3 = t % d3;
                        const int kx = min(kxg + xt * Q + q, Nx - 1);
                        const int ox = kx <= (Nx >> 1) ? kx : Nx - kx;
                        const float* f1 = sv.fac[m][0] + (int64_t)ox * d1;
                        float acc = 0.f;
                        for (int cc1 = 0; cc1 < d1; ++cc1) acc = fmaf(G[c3 * d1 + cc1], __ldg(&f1[cc1]), acc);
                        H[t] = acc;
                    }
                    __syncthreads();
                    for (int t = tid; t < NK * Q; t += NT) {
                        const int kh = t / Q, q = t % Q;
                        const float* f3 = sv.fac[m][2] + (int64_t)kh * d3;
                        float acc = 0.f;
                        for (int c3 = 0; c3 < d3; ++c3) acc = fmaf(H[q * d3 + c3], __ldg(&f3[c3]), acc);
                        KV0[(m * NK + kh) * Q + q] = acc;
                    }
                }
            }
        }
        const float* KV = tucker ? KV0 : KV0 + ((s / nrhs) & 1) * (P::KV_b / sizeof(float));
        mbar_wait(&bar[st], (uint32_t)((s >> 1) & 1));
        // forward level 1 (thread (c, n2, q)): FFT_R1 over n1 of x[R2 n1 + n2], twiddle W_N^{n2 k1}
        if (tid < NT1) {
            float2 v[R1];
#pragma unroll
            for (int n1 = 0; n1 < R1; ++n1) {
                const int z = R2 * n1 + n2;
                v[n1] = (n1 < R1 / 2 && pok[z]) ? slot[(c1 * NH + z) * Q + q1] : zero;
            }
            reg_fft<R1, -1, true>(v);
#pragma unroll
            for (int k = 1; k < R1; ++k) v[k] = cmul(v[k], tws[n2 * k]);
#pragma unroll
            for (int k = 0; k < R1; ++k) T[c1 * EM + P::ti(n2, k, q1)] = v[k];
        }
        __syncthreads();
        if (tid == 0) {   // the other slot: its output store (previous tile) must have left smem
            tma_store_wait_read0();
            issue(s + 1, st ^ 1);
        }
        // level 2 (thread (k1, q)): forward FFT_R2 of all 5 components -> kz = k1 + R1 k2,
        // MAC in registers, inverse FFT_R2, twiddle W_N^{-n2 k1}, back to the same elements
        if (tid < NT2) {
            const int kx = kxg + xt * Q + q2;
            const float gx = kx <= (Nx >> 1) ? g : -g, gy = ky <= (Ny >> 1) ? g : -g;
            float2 u[5][R2];
#pragma unroll
            for (int c = 0; c < 5; ++c) {
#pragma unroll
                for (int m = 0; m < R2; ++m) u[c][m] = T[c * EM + P::ti(m, k1, q2)];
                reg_fft<R2, -1>(u[c]);
            }
#pragma unroll
            for (int k2 = 0; k2 < R2; ++k2) {
                const int kz = k1 + R1 * k2;
                const int kh = kz <= NH ? kz : N - kz;
                const float s3 = kz <= NH ? 1.f : -1.f;   // K1z is odd in kz
                const float* kp = KV + kh * Q + q2;
                const float f0 = g * kp[0 * NK * Q], f1 = gx * kp[1 * NK * Q], f2 = gy * kp[2 * NK * Q];
                const float f3 = (-2.f * g) * s3 * kp[3 * NK * Q];
                const float f4 = g * kp[4 * NK * Q], f5 = g * kp[5 * NK * Q], f6 = (4.f * g) * kp[6 * NK * Q];
                const float2 Ix = u[0][k2], Iy = u[1][k2], Iz = u[2][k2], I2 = u[3][k2], I3 = u[4][k2];
                const float2 m1x = cadd(I2, I3), m1y = csub(I3, I2);
                const float2 Qx = cfma_s(Ix, -f1, cmul_i(m1x, f4));
                const float2 Qy = cfma_s(Iy, -f2, cmul_i(m1y, f5));
                const float2 Qz = cfma_s(Iz, -f3, cmul_i(I3, f6));
                u[0][k2] = cfma_s(m1x, f1, cmul_i(Ix, f0));
                u[1][k2] = cfma_s(m1y, f2, cmul_i(Iy, f0));
                u[2][k2] = cfma_s(I3, f3, cmul_i(Iz, f0));
                u[3][k2] = csub(Qx, Qy);
                u[4][k2] = cadd(cadd(Qx, Qy), Qz);
            }
#pragma unroll
            for (int c = 0; c < 5; ++c) {
                reg_fft<R2, +1>(u[c]);
#pragma unroll
                for (int m = 0; m < R2; ++m) {
                    float2 w = tws[m * k1];
                    w.y = -w.y;
                    T[c * EM + P::ti(m, k1, q2)] = m ? cmul(u[c][m], w) : u[c][m];
                }
            }
        }
        __syncthreads();
        // inverse level 2 (thread (c, n2, q)): IFFT_R1 over k1 -> z = n2 + R2 n1, cropped to z < Kz
        if (tid < NT1) {
            float2 v[R1];
#pragma unroll
            for (int k = 0; k < R1; ++k) v[k] = T[c1 * EM + P::ti(n2, k, q1)];
            reg_fft<R1, +1>(v);
#pragma unroll
            for (int n1 = 0; n1 < R1 / 2; ++n1) {
                const int z = n2 + R2 * n1;
                if (z < Kz) slot[(c1 * NH + z) * Q + q1] = v[n1];
            }
        }
        fence_proxy_async_smem();
        __syncthreads();
        if (tid == 0) {
#pragma unroll
            for (int c = 0; c < 5; ++c) tma_store_3d(&tmap, xt * Q, ky, (r * 5 + c) * Kz, slot + c * NH * Q);
            tma_store_commit();
        }
    }
    if (tid == 0) tma_store_wait0();
}

// ---------------------------------------------------------------------------
// host-side dispatch
namespace {

template <typename F>
void prep(F* kern, size_t bytes) {
    // every pass kernel gets the max shared-memory carveout; >48 KB needs opt-in.  The attributes
    // are set once per (kernel, size): these driver calls cost host time on every launch otherwise.
    static thread_local std::vector<std::pair<const void*, size_t>> done;
    for (const auto& d : done)
        if (d.first == (const void*)kern && d.second >= bytes) return;
    SVH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                  (int)cudaSharedmemCarveoutMaxShared));
    if (bytes > 48 * 1024)
        SVH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    done.emplace_back((const void*)kern, bytes);
}

// rows per CTA for the row passes (A/E)
template <int N>
constexpr int row_q() {
    // N >= 2048: the 64-point first level needs ~170 registers per thread; one row (64 threads)
    // per CTA lets several CTAs share an SM and overlap one's loads with the others' barriers
    // (measured on 1024^2 grids: 4 rows/CTA A 7.4 / E 11.3 ms, 2 rows 5.0 / 7.5, 1 row 4.8 / 6.8)
    return fft_r2(N) == 1 ? 128 : N >= 2048 ? 1 : (256 / fft_threads_per_pencil(N) > 0 ? 256 / fft_threads_per_pencil(N) : 1);
}
// pencils per CTA for the strided passes (B/D)
template <int N>
constexpr int col_q() {
    return fft_r2(N) == 1 ? 128 : (fft_r1(N) >= 64 ? 4 : 8);
}

}  // namespace
// Geometry of one pass invocation: the whole grid, or one slab of the slab-decomposed
// matvec: x-slab passes B-D see the array columns kx0 .. kx0+nx-1 of the
// global embedding; row passes A/E see the y rows y0 .. y0+kyl-1 of every plane.
struct Geom {
    int nx;                   // x extent of the X1 / X2 arrays
    int kx0;                  // global kx of array column 0
    int kyl, y0;              // rows of the row passes
    const int32_t* rowlist;   // pass A: non-empty global rows z*Ky + y (ascending)
    int nrows;
};
static Geom whole_grid(const svh_handle* h) {
    return Geom{h->nx, 0, h->ky, 0, h->d_rowlist, (int)h->n_rows_ne};
}
namespace {

// persistent grid size for a kernel: min(work units, SMs x resident CTAs)
// (occupancy queried once per (device, kernel, block, smem): the query costs host time)
template <typename F>
int persistent_grid(F kern, int nt, size_t smem, int64_t units) {
    struct Rec {
        int dev;
        const void* k;
        int nt;
        size_t smem;
        int ctas;
    };
    static thread_local std::vector<Rec> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    int ctas = 0;
    for (const auto& r : cache)
        if (r.dev == dev && r.k == (const void*)kern && r.nt == nt && r.smem == smem) ctas = r.ctas;
    if (ctas == 0) {
        int nsm = 148, occ = 1;
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, nt, smem);
        ctas = nsm * std::max(occ, 1);
        cache.push_back(Rec{dev, (const void*)kern, nt, smem, ctas});
    }
    return (int)std::max<int64_t>(1, std::min<int64_t>(units, ctas));
}

template <int N>
void run_pass_a(svh_handle* h, const Geom& g, const float2* in, float2* X1, bool packed, int nrhs, cudaStream_t s) {
    const int rows = g.kyl * h->kz;
    const int64_t Ktl = (int64_t)g.kyl * h->kz * h->kx;
    if constexpr (N >= 128) {
        using PL = RowPlan<N>;
        const int nlist = g.nrows;
        if (nlist == 0) return;
        const int64_t units = (int64_t)((nlist + PL::RPC - 1) / PL::RPC) * 5 * nrhs;
        const size_t smem = PL::smem + (size_t)PL::RPC * 2 * RowSlot<N>::A_b;
        auto go = [&](auto kern) {
            prep(kern, smem);
            SVH_LAUNCH(kern, persistent_grid(kern, PL::NT, smem, units), PL::NT, smem, s, in, X1,
                       h->d_rowinfo, h->rowW, g.rowlist, nlist, h->d_tw[0], h->kx, rows, h->K, Ktl, h->ky, g.kyl,
                       g.y0, 5 * nrhs);
        };
        if (packed)
            go(k_rowA<N, true>);
        else
            go(k_rowA<N, false>);
        return;
    }
    constexpr int Q = row_q<N>();
    const int nt = fft_threads_per_pencil(N) * Q;
    const size_t smem = fft_r2(N) == 1 ? 0 : (size_t)Q * (N + N / fft_r1(N)) * sizeof(float2);
    const int nlist = g.nrows;
    if (nlist == 0) return;
    dim3 grid((nlist + Q - 1) / Q, 5 * nrhs);
    if (packed) {
        prep(k_row_fwd<N, Q, true>, smem);
        SVH_LAUNCH((k_row_fwd<N, Q, true>), grid, nt, smem, s, in, X1, h->d_rowinfo, h->rowW, g.rowlist, nlist,
                   h->d_tw[0], h->kx, rows, h->K, Ktl, h->ky, g.kyl, g.y0);
    } else {
        prep(k_row_fwd<N, Q, false>, smem);
        SVH_LAUNCH((k_row_fwd<N, Q, false>), grid, nt, smem, s, in, X1, h->d_rowinfo, h->rowW, g.rowlist, nlist,
                   h->d_tw[0], h->kx, rows, h->K, Ktl, h->ky, g.kyl, g.y0);
    }
}

template <int N, int DIR>
void run_pass_y(svh_handle* h, const Geom& g, const float2* in, float2* out, int Lin, int Lout, int nrhs,
                cudaStream_t s) {
    const int nx = g.nx;
    if constexpr (N == 2048) {
        // 2048-point pencils: Stockham radix-16, TMA-staged input, TMA-stored output (B)
        // (ypass.cuh).  For N <= 1024, k_ytma measured faster (cfg4 B/D 3.2/2.4 vs 4.2/3.1 ms).
        constexpr int Q = 4;
        using P = YPlan<N, Q, DIR>;
        CUtensorMap tin, tout;
        const int rows_in = DIR < 0 ? h->ky : h->ny;
        const float2* x2 = DIR < 0 ? out : in;   // the X2 side of the pass
        if (nx % Q == 0 &&
            encode_tmap_c64_3d(&tin, in, (uint64_t)nx, (uint64_t)rows_in, (uint64_t)5 * nrhs * h->kz, (uint64_t)nx,
                               (uint64_t)nx * rows_in, Q, P::BOX) &&
            encode_tmap_c64_3d(&tout, x2, (uint64_t)nx, (uint64_t)h->ny, (uint64_t)5 * nrhs * h->kz, (uint64_t)nx,
                               (uint64_t)nx * h->ny, Q, P::BOX)) {
            const int tiles_x = nx / Q;
            const int ntiles = tiles_x * h->nzp * 5 * nrhs;
            auto kern = k_ypass<N, Q, DIR>;
            prep(kern, P::smem);
            SVH_LAUNCH(kern, persistent_grid(kern, P::NT, P::smem, ntiles), P::NT, P::smem, s, out, tin, tout,
                       h->d_tw[1], nx, h->kz, Lin, Lout, ntiles, tiles_x, h->d_planes, h->nzp, h->d_rowmask,
                       h->rowMW);
            return;
        }
    }
    if constexpr (N >= 128 && N <= 2048) {
        // TMA ring / TMA-stored tiles of 4 pencils (k_ytma)
        constexpr int QQ = 4;
        using P = YTma<N, DIR, 2, QQ>;
        CUtensorMap tmap;
        const float2* x2 = DIR < 0 ? out : in;   // the X2 side of the pass
        if (nx % QQ == 0 && encode_tmap_c64_3d(&tmap, x2, (uint64_t)nx, (uint64_t)h->ny, (uint64_t)5 * nrhs * h->kz,
                                               (uint64_t)nx, (uint64_t)nx * h->ny, QQ, P::BOX)) {
            const int tiles_x = nx / QQ;
            const int ntiles = tiles_x * h->nzp * 5 * nrhs;
            auto kern = k_ytma<N, DIR, 2, QQ>;
            prep(kern, P::smem);
            SVH_LAUNCH(kern, persistent_grid(kern, P::NT, P::smem, ntiles), P::NT, P::smem, s, in, out, tmap,
                       h->d_tw[1], nx, h->kz, Lin, Lout, ntiles, tiles_x, h->d_planes, h->nzp, h->d_rowmask,
                       h->rowMW);
            return;
        }
    }
    // generic one-tile-per-CTA pass: N <= 64 (one thread per pencil), N = 4096, and grids whose
    // x extent does not tile (tested by the max-extent and tiny-grid parity tests)
    constexpr int Q = col_q<N>();
    const int nt = fft_threads_per_pencil(N) * Q;
    const size_t smem = fft_r2(N) == 1 ? 0 : (size_t)em_size<N, Q>() * sizeof(float2);
    dim3 grid((nx + Q - 1) / Q, h->nzp, 5 * nrhs);
    prep(k_col<N, Q, DIR>, smem);
    SVH_LAUNCH((k_col<N, Q, DIR>), grid, nt, smem, s, in, out, h->d_tw[1], nx, h->kz, Lin, Lout, h->d_planes,
               h->d_rowmask, h->rowMW);
}

// k_ztma2 launch: false if the grid does not tile (x extent not a multiple of Q) or the
// tensor map cannot be encoded (the caller then takes another pass-C kernel)
template <int N, int Q2, int R2>
bool launch_ztma2(svh_handle* h, const Geom& g, float2* X2, int nrhs, const SpecView& sv, cudaStream_t s) {
    using P2 = ZTma2<N, Q2, R2>;
    CUtensorMap tm2;
    if (g.nx % Q2 != 0 ||
        !encode_tmap_c64_3d_box(&tm2, X2, (uint64_t)g.nx, (uint64_t)h->ny, (uint64_t)5 * nrhs * h->kz, (uint64_t)g.nx,
                                (uint64_t)g.nx * h->ny, Q2, 1, (uint32_t)h->kz))
        return false;
    const int tiles_x = g.nx / Q2;
    const int ngroups = tiles_x * h->ny;
    int dev = 0, nsm = 148, occ = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    prep(k_ztma2<N, Q2, R2>, P2::smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_ztma2<N, Q2, R2>, P2::NT, P2::smem);
    SVH_LAUNCH((k_ztma2<N, Q2, R2>), std::min(ngroups, nsm * std::max(occ, 1)), P2::NT, P2::smem, s, tm2, sv,
               h->d_tw[2], h->nx, h->ny, h->kz, h->gscale, nrhs, ngroups, tiles_x, h->d_planeok, g.kx0);
    return true;
}

template <int N>
void run_pass_c(svh_handle* h, const Geom& g, float2* X2, int nrhs, cudaStream_t s) {
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
    if constexpr (N >= 64 && N <= 256) {
        // 16 kx per tile: pass C's HBM pattern is Q*8-byte runs at the plane stride; a pure
        // read-modify-write of that pattern reaches 2.4 / 4.2 / 5.4 TB/s for Q = 8 / 16 / 32
        // (scripts/micro/zpattern.cu on B200), so the tile is as wide as shared memory allows
        // (Q = 8 when high Tucker ranks leave no room for 16)
        int dmax = 0;
        if (h->use_tucker)
            for (int m = 0; m < 7; ++m)
                for (int a = 0; a < 3; ++a) dmax = std::max(dmax, sv.rk[m][a]);
        const bool fits = dmax <= kTuckerMaxRank;
        // plans: (R2, Q, threads): every thread runs TL1 = 5 R2 Q / threads L1 tasks and at most one
        // L2 task.  Dense spectra: T double-buffered; Tucker: one T buffer, the freed shared memory
        // holds the mode-3 factor rows and the expansion scratch (rank bucket 16 / 32)
        auto launch = [&](auto R2c, auto Qc, auto NTc) -> bool {
            constexpr int R2 = decltype(R2c)::value, Q = decltype(Qc)::value, NT = decltype(NTc)::value;
            using P = ZPlan<N, R2, Q, NT>;
            if (g.nx % Q != 0 || !fits) return false;
            const int64_t units = (int64_t)(h->ny / 2 + 1) * (g.nx / Q);
            auto go = [&](auto kern, size_t smem) -> bool {
                if (smem > 227 * 1024) return false;
                prep(kern, smem);
                SVH_LAUNCH(kern, persistent_grid(kern, NT, smem, units), NT, smem, s, X2, sv, h->d_tw[2], h->nx,
                           h->ny, h->kz, g.nx, g.kx0, h->gscale, nrhs, h->d_planeok);
                return true;
            };
            if (!h->use_tucker)
                return go(k_zpass<N, R2, Q, NT, 2, 0>, P::smem(2, 0)) || go(k_zpass<N, R2, Q, NT, 1, 0>, P::smem(1, 0));
            if (dmax <= 16) return go(k_zpass<N, R2, Q, NT, 1, 16>, P::smem(1, 16));
            return go(k_zpass<N, R2, Q, NT, 1, 32>, P::smem(1, 32));
        };
        if constexpr (N == 128) {
            if (launch(std::integral_constant<int, 8>{}, std::integral_constant<int, 16>{},
                       std::integral_constant<int, 320>{}) ||
                launch(std::integral_constant<int, 8>{}, std::integral_constant<int, 8>{},
                       std::integral_constant<int, 160>{}))
                return;
        } else if constexpr (N == 64) {
            if (launch(std::integral_constant<int, 4>{}, std::integral_constant<int, 16>{},
                       std::integral_constant<int, 320>{}) ||
                launch(std::integral_constant<int, 4>{}, std::integral_constant<int, 8>{},
                       std::integral_constant<int, 160>{}))
                return;
        } else {   // N == 256
            if (launch(std::integral_constant<int, 8>{}, std::integral_constant<int, 8>{},
                       std::integral_constant<int, 320>{}) ||
                launch(std::integral_constant<int, 8>{}, std::integral_constant<int, 4>{},
                       std::integral_constant<int, 160>{}))
                return;
        }
    }
    if constexpr (N >= 2 && N <= 32) {
        // one thread per (component, pencil) z-FFT in registers, 32 pencils x 5 components per CTA
        dim3 grid((g.nx + 31) / 32, h->ny);
        if (sv.spec) {
            const size_t smem2 = zmac2_smem<N>();
            prep(k_zmac2<N>, smem2);
            SVH_LAUNCH((k_zmac2<N>), grid, 160, smem2, s, X2, sv, h->nx, h->ny, h->kz, h->gscale, nrhs,
                       (uint64_t)h->planemask, g.nx, g.kx0);
        } else {
            const size_t smem = zmac_smem<N>();
            prep(k_zmac<N>, smem);
            SVH_LAUNCH((k_zmac<N>), grid, 160, smem, s, X2, sv, h->nx, h->ny, h->kz, h->gscale, nrhs,
                       (uint64_t)h->planemask, g.nx, g.kx0, 1);
        }
        return;
    }
    if constexpr (N == 512) {
        if (launch_ztma2<512, 4, 8>(h, g, X2, nrhs, sv, s)) return;
    }
    if constexpr (N <= 64) {
        // N = 1 and x extents that do not tile k_zpass: one thread per (component, pencil)
        constexpr int Q = N >= 64 ? 16 : 32;
        const size_t smem = freq_small_smem<N, Q, false>();
        dim3 grid((g.nx + Q - 1) / Q, h->ny);
        prep(k_freq_small<N, Q, false>, smem);
        SVH_LAUNCH((k_freq_small<N, Q, false>), grid, 5 * Q, smem, s, X2, sv, h->nx, h->ny, h->kz, h->gscale, nrhs,
                   (uint64_t)h->planemask, g.nx, g.kx0);
    } else {
        // generic shared-memory z pass: N >= 1024 and x extents that do not tile
        const int tpp = fft_threads_per_pencil(N);
        int Q = std::min(8, std::max(1, fft_max_threads(N) / (tpp * 5)));   // <= 8: Tucker H tile
        while (Q > 1 && (size_t)N * (5 * Q + 1) * sizeof(float2) > 160 * 1024) Q >>= 1;
        const int nt = std::max(32, tpp * 5 * Q);
        const size_t smem = (size_t)N * (5 * Q + 1) * sizeof(float2);
        dim3 grid((g.nx + Q - 1) / Q, h->ny, nrhs);
        prep(k_freq_big<N>, smem);
        SVH_LAUNCH((k_freq_big<N>), grid, nt, smem, s, X2, sv, h->d_tw[2], h->nx, h->ny, h->kz, Q, h->gscale,
                   h->d_planeok, g.nx, g.kx0);
    }
}

template <int N>
void run_pass_e(svh_handle* h, const Geom& g, const float2* X1, const float2* in, float2* out, bool packed,
                bool green_only,
                int nrhs, cudaStream_t s) {
    const int rows = g.kyl * h->kz;
    const int64_t Ktl = (int64_t)g.kyl * h->kz * h->kx;
    const int nzl = (int)h->mats.size() + 1;
    // packed output: only the non-empty rows; grid output: every row (empty ones get zeros)
    const int nlist = packed ? (int)h->n_rows_ne : rows;
    const int32_t* rl = packed ? h->d_rowlist : nullptr;
    if constexpr (N >= 128) {
        using PL = RowPlan<N>;
        if (nlist == 0) return;
        const int64_t units = (int64_t)((nlist + PL::RPC - 1) / PL::RPC) * 5 * nrhs;
        const size_t smem = (size_t)PL::RPC * RowSlotE<N>::G_b;
        auto go = [&](auto kern) {
            prep(kern, smem);
            SVH_LAUNCH(kern, persistent_grid(kern, PL::NT, smem, units), PL::NT, smem, s, X1, out, in,
                       h->d_rowinfo, h->rowW, rl, nlist, h->d_rowmask, h->rowMW, h->ky, h->d_matp, h->d_zloc, nzl,
                       h->d_tw[0], h->kx, rows, h->K, Ktl, (int)green_only, g.kyl, g.y0, 5 * nrhs);
        };
        if (packed)
            go(k_rowE<N, true>);
        else
            go(k_rowE<N, false>);
        return;
    }
    constexpr int Q = row_q<N>();
    const int nt = fft_threads_per_pencil(N) * Q;
    const size_t smem = fft_r2(N) == 1 ? 0 : (size_t)Q * (N + N / fft_r1(N)) * sizeof(float2);
    dim3 grid((nlist + Q - 1) / Q, 5 * nrhs);
    if (packed) {
        prep(k_row_inv<N, Q, true>, smem);
        SVH_LAUNCH((k_row_inv<N, Q, true>), grid, nt, smem, s, X1, out, in, h->d_rowinfo, h->rowW, rl, nlist,
                   h->d_rowmask, h->rowMW, h->ky, h->d_matp, h->d_zloc, nzl, h->d_tw[0], h->kx, rows, h->K, Ktl,
                   (int)green_only, g.kyl, g.y0);
    } else {
        prep(k_row_inv<N, Q, false>, smem);
        SVH_LAUNCH((k_row_inv<N, Q, false>), grid, nt, smem, s, X1, out, in, h->d_rowinfo, h->rowW, rl, nlist,
                   h->d_rowmask, h->rowMW, h->ky, h->d_matp, h->d_zloc, nzl, h->d_tw[0], h->kx, rows, h->K, Ktl,
                   (int)green_only, g.kyl, g.y0);
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
    size_t budget = (size_t)(0.75 * (double)(fr + (size_t)h->ws_rhs * per));
    return (int)std::max<size_t>(1, std::min<size_t>(64, budget / per));
}

// one sub-batch of nr RHS on stream s with workspace slices X1, X2
static void matvec_batch(svh_handle* h, const float2* in, float2* out, float2* X1, float2* X2, int nr,
                         bool green_only, bool packed, cudaStream_t s, int plan) {
    // SVH_SYNC_DEBUG (debugging aid, include/svh.h): synchronise after every pass and report the
    // failing pass; it does not change which kernels run
    static const bool dbg = getenv("SVH_SYNC_DEBUG") != nullptr;
    auto tick = [&](int pass, bool begin) {
        if (dbg && !begin) {
            cudaError_t e = cudaStreamSynchronize(s);
            if (e != cudaSuccess)
                throw Error{SVH_ECUDA, "pass " + std::to_string(pass) + ": " + cudaGetErrorString(e)};
        }
        if (!h->prof_on) return;
        if (begin) {
            svh_handle::ProfRec r{pass, nullptr, nullptr};
            SVH_CUDA(cudaEventCreate(&r.a));
            SVH_CUDA(cudaEventCreate(&r.b));
            SVH_CUDA(cudaEventRecord(r.a, s));
            h->prof.push_back(r);
        } else {
            SVH_CUDA(cudaEventRecord(h->prof.back().b, s));
        }
    };
    if (plan == 3) {
        // plan P3s (p3s.cu): x | fused y-z-y on chip | x, profiled as one record (pass 5)
        tick(5, true);
        p3s_matvec(h, in, out, X1, nr, green_only, packed, s);
        tick(5, false);
        return;
    }
    const Geom g = whole_grid(h);
    tick(0, true);
    SVH_DISPATCH_N(h->nx, run_pass_a<NN>(h, g, in, X1, packed, nr, s));
    tick(0, false);
    tick(1, true);
    SVH_DISPATCH_N(h->ny, (run_pass_y<NN, -1>(h, g, X1, X2, h->ky, h->ny, nr, s)));
    tick(1, false);
    tick(2, true);
    SVH_DISPATCH_N(h->nz, run_pass_c<NN>(h, g, X2, nr, s));
    tick(2, false);
    tick(3, true);
    SVH_DISPATCH_N(h->ny, (run_pass_y<NN, +1>(h, g, X2, X1, h->ny, h->ky, nr, s)));
    tick(3, false);
    tick(4, true);
    SVH_DISPATCH_N(h->nx, run_pass_e<NN>(h, g, X1, in, out, packed, green_only, nr, s));
    tick(4, false);
}

int choose_plan(svh_handle* h, const float2* in, float2* out, int nr, bool green_only, bool packed,
                cudaStream_t s);

void matvec(svh_handle* h, const float2* I, float2* CC, int nrhs, bool green_only, bool packed, cudaStream_t s) {
    // RHS chunks sized to the workspace budget (max_chunk) and balanced (8 RHS with room for 7
    // run as 4 + 4, not 7 + 1); every pass fills the GPU on its own, so the chunks run back to
    // back on the caller's stream
    const int maxc = std::max(1, std::min(nrhs, max_chunk(h)));
    const int nch = (nrhs + maxc - 1) / maxc;
    const int chunk = (nrhs + nch - 1) / nch;
    ensure_workspace(h, chunk);
    const int64_t per_rhs = 5 * (packed ? h->K : h->Kt);
    for (int r0 = 0; r0 < nrhs; r0 += chunk) {
        const int nr = std::min(chunk, nrhs - r0);
        const int plan = choose_plan(h, I + r0 * per_rhs, CC + r0 * per_rhs, nr, green_only, packed, s);
        matvec_batch(h, I + r0 * per_rhs, CC + r0 * per_rhs, h->X1, h->X2, nr, green_only, packed, s, plan);
        h->last_plan = plan;
    }
}

// Plan for a chunk of nr RHS (SURVEY 8(d) reporting rule: plans are chosen by absolute time).
// opts.plan = 5 / 3 forces P5 / P3s; auto (0) takes P5 unless P3s is eligible (thin grid,
// p3s_eligible), and then times both once per chunk size on the caller's data (two warm runs
// of each, then one timed run of each; the last run is P3s, so CC holds a valid product
// either way) and keeps the faster.  Not while the stream is being captured into a graph.
int choose_plan(svh_handle* h, const float2* in, float2* out, int nr, bool green_only, bool packed, cudaStream_t s) {
    if (h->opts.plan == 5) return 5;
    if (h->opts.plan == 3) {
        SVH_CHECK(p3s_eligible(h), SVH_EINVAL, "plan P3s needs Nz <= 8, 128 <= Nx <= 1024, Ny <= 1024 and a "
                                               "y-z slab that fits shared memory");
        return 3;
    }
    if (!p3s_eligible(h)) return 5;
    for (const auto& t : h->plan_tuned)
        if (t.first == nr) return t.second;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    SVH_CUDA(cudaStreamIsCapturing(s, &cs));
    if (cs != cudaStreamCaptureStatusNone) return 3;
    const bool prof = h->prof_on;
    h->prof_on = false;
    cudaEvent_t ev[4];
    for (auto& e : ev) SVH_CUDA(cudaEventCreate(&e));
    for (int w = 0; w < 2; ++w) {
        matvec_batch(h, in, out, h->X1, h->X2, nr, green_only, packed, s, 5);
        matvec_batch(h, in, out, h->X1, h->X2, nr, green_only, packed, s, 3);
    }
    SVH_CUDA(cudaEventRecord(ev[0], s));
    matvec_batch(h, in, out, h->X1, h->X2, nr, green_only, packed, s, 5);
    SVH_CUDA(cudaEventRecord(ev[1], s));
    SVH_CUDA(cudaEventRecord(ev[2], s));
    matvec_batch(h, in, out, h->X1, h->X2, nr, green_only, packed, s, 3);
    SVH_CUDA(cudaEventRecord(ev[3], s));
    SVH_CUDA(cudaEventSynchronize(ev[3]));
    float t5 = 0.f, t3 = 0.f;
    SVH_CUDA(cudaEventElapsedTime(&t5, ev[0], ev[1]));
    SVH_CUDA(cudaEventElapsedTime(&t3, ev[2], ev[3]));
    for (auto& e : ev) cudaEventDestroy(e);
    h->prof_on = prof;
    const int plan = t3 <= t5 ? 3 : 5;
    h->plan_tuned.push_back({nr, plan});
    h->plan_ms.push_back({t5, t3});
    return plan;
}

// ---------------------------------------------------------------------------
// Slab-decomposed matvec: P ranks; rank r holds the y-slab
// y in [r Kyl, (r+1) Kyl) of every plane (grid layout), Kyl = Ky/P.
//   forward : pass A on the slab's rows, pack X1 by destination kx-slab        -> send
//   (all-to-all #1: every rank now has kx in [r Nxl, (r+1) Nxl) for all y, Nxl = Nx/P)
//   middle  : unpack, passes B, C, D on the kx-slab (global kx offset for the kernels),
//             pack by destination y-slab                                         -> send
//   (all-to-all #2)
//   backward: unpack, pass E on the slab's rows (+ local term)                   -> CC
// All-to-all buffers: [peer p][5 nrhs Kz][Kyl][Nxl] complex64 (equal chunks).  Only the
// minimum volume is exchanged: the x-FFT'd current, 2 Kt points/comp per direction.
namespace {
// element (p, b, y, k) of the buffer [p][b][y][k] <-> array element b*SB + y*SY + p*SP + k
__global__ void k_slab_copy(float2* __restrict__ buf, float2* __restrict__ arr, int P, int64_t Bt, int Kyl, int Nxl,
                            int64_t SB, int64_t SY, int64_t SP, int to_array) {
    const int64_t total = (int64_t)P * Bt * Kyl * Nxl;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(i % Nxl);
        int64_t r = i / Nxl;
        const int y = (int)(r % Kyl);
        r /= Kyl;
        const int64_t b = r % Bt;
        const int p = (int)(r / Bt);
        const int64_t a = b * SB + (int64_t)y * SY + (int64_t)p * SP + k;
        if (to_array)
            arr[a] = buf[i];
        else
            buf[i] = arr[a];
    }
}

void slab_copy(float2* buf, float2* arr, int P, int64_t Bt, int Kyl, int Nxl, int64_t SB, int64_t SY, int64_t SP,
               bool to_array, cudaStream_t s) {
    const int64_t total = (int64_t)P * Bt * Kyl * Nxl;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int grid = (int)std::min<int64_t>((total + 255) / 256, (int64_t)nsm * 8);
    SVH_LAUNCH(k_slab_copy, std::max(grid, 1), 256, 0, s, buf, arr, P, Bt, Kyl, Nxl, SB, SY, SP, (int)to_array);
}

void check_slab(const svh_handle* h, int rank, int P) {
    SVH_CHECK(P >= 1 && rank >= 0 && rank < P, SVH_EINVAL, "bad slab rank / count");
    SVH_CHECK(h->ky % P == 0 && h->nx % P == 0, SVH_EINVAL, "slab decomposition needs Ky % P == 0 and Nx % P == 0");
}

const svh_handle::SlabRows& slab_rows(svh_handle* h, int rank, int P) {
    for (auto& sr : h->slab_rows)
        if (sr.P == P && sr.rank == rank) return sr;
    const int Kyl = h->ky / P, y0 = rank * Kyl;
    std::vector<int32_t> rl;
    for (int32_t row : h->h_rowlist) {
        const int y = row % h->ky;
        if (y >= y0 && y < y0 + Kyl) rl.push_back(row);
    }
    svh_handle::SlabRows sr{P, rank, nullptr, (int)rl.size()};
    if (!rl.empty()) {
        SVH_CUDA(cudaMalloc(&sr.d, rl.size() * sizeof(int32_t)));
        SVH_CUDA(cudaMemcpy(sr.d, rl.data(), rl.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    }
    h->slab_rows.push_back(sr);
    return h->slab_rows.back();
}
}  // namespace

void slab_sizes(const svh_handle* h, int P, int64_t* out4) {
    check_slab(h, 0, P);
    const int64_t Kyl = h->ky / P, Nxl = h->nx / P;
    out4[0] = Kyl;
    out4[1] = Nxl;
    out4[2] = 5 * (int64_t)h->kz * Kyl * Nxl;       // complex elements per peer chunk per RHS
    out4[3] = out4[2] * P;                          // send / recv buffer elements per RHS
}

// pass A on the slab's rows -> X1 [b][y][Nx] (the part of slab_forward before the pack)
void slab_forward_compute(svh_handle* h, int rank, int P, const float2* I, int nrhs, cudaStream_t s) {
    check_slab(h, rank, P);
    ensure_workspace(h, nrhs);
    const int Kyl = h->ky / P;
    const auto& sr = slab_rows(h, rank, P);
    const Geom g{h->nx, 0, Kyl, rank * Kyl, sr.d, sr.n};
    SVH_DISPATCH_N(h->nx, run_pass_a<NN>(h, g, I, h->X1, false, nrhs, s));
}

// unpack recv [s][b][y][k] -> X1 [b][s Kyl + y][k], passes B, C, D on the kx-slab (X1 in place)
void slab_middle_compute(svh_handle* h, int rank, int P, const float2* recv, int nrhs, cudaStream_t s) {
    check_slab(h, rank, P);
    ensure_workspace(h, nrhs);
    const int Kyl = h->ky / P, Nxl = h->nx / P;
    const int64_t Bt = 5LL * nrhs * h->kz;
    slab_copy(const_cast<float2*>(recv), h->X1, P, Bt, Kyl, Nxl, (int64_t)h->ky * Nxl, Nxl, (int64_t)Kyl * Nxl, true,
              s);
    const Geom g{Nxl, rank * Nxl, h->ky, 0, nullptr, 0};
    SVH_DISPATCH_N(h->ny, (run_pass_y<NN, -1>(h, g, h->X1, h->X2, h->ky, h->ny, nrhs, s)));
    SVH_DISPATCH_N(h->nz, run_pass_c<NN>(h, g, h->X2, nrhs, s));
    SVH_DISPATCH_N(h->ny, (run_pass_y<NN, +1>(h, g, h->X2, h->X1, h->ny, h->ky, nrhs, s)));
}

void slab_forward(svh_handle* h, int rank, int P, const float2* I, float2* send, int nrhs, cudaStream_t s) {
    slab_forward_compute(h, rank, P, I, nrhs, s);
    const int Kyl = h->ky / P, Nxl = h->nx / P;
    const int64_t Bt = 5LL * nrhs * h->kz;
    slab_copy(send, h->X1, P, Bt, Kyl, Nxl, (int64_t)Kyl * h->nx, h->nx, Nxl, false, s);
}

void slab_middle(svh_handle* h, int rank, int P, const float2* recv, float2* send, int nrhs, cudaStream_t s) {
    slab_middle_compute(h, rank, P, recv, nrhs, s);
    const int Kyl = h->ky / P, Nxl = h->nx / P;
    const int64_t Bt = 5LL * nrhs * h->kz;
    slab_copy(send, h->X1, P, Bt, Kyl, Nxl, (int64_t)h->ky * Nxl, Nxl, (int64_t)Kyl * Nxl, false, s);
}

void slab_backward(svh_handle* h, int rank, int P, const float2* recv, const float2* I, float2* CC, int nrhs,
                   bool green_only, cudaStream_t s) {
    check_slab(h, rank, P);
    ensure_workspace(h, nrhs);
    const int Kyl = h->ky / P, Nxl = h->nx / P;
    const int64_t Bt = 5LL * nrhs * h->kz;
    // [s][b][y][k] -> X1 [b][y][s Nxl + k]
    slab_copy(const_cast<float2*>(recv), h->X1, P, Bt, Kyl, Nxl, (int64_t)Kyl * h->nx, h->nx, Nxl, true, s);
    const Geom g{h->nx, 0, Kyl, rank * Kyl, nullptr, 0};
    SVH_DISPATCH_N(h->nx, run_pass_e<NN>(h, g, h->X1, I, CC, false, green_only, nrhs, s));
}

// ---------------------------------------------------------------------------
// Host-buffer matvec (svh_matvec_host): the RHS stream through the GPU in chunks; the H2D
// copy of chunk c+1 and the D2H copy of chunk c-1 run on their own streams while chunk c is
// multiplied, so the host<->device traffic hides behind the passes (pinned host memory).
void free_host_pipe(svh_handle* h) {
    auto* P = h->pipe;
    if (!P) return;
    for (int k = 0; k < 2; ++k) {
        cudaFree(P->din[k]);
        cudaFree(P->dout[k]);
        if (P->in_ready[k]) cudaEventDestroy(P->in_ready[k]);
        if (P->mv_done[k]) cudaEventDestroy(P->mv_done[k]);
        if (P->out_done[k]) cudaEventDestroy(P->out_done[k]);
    }
    if (P->h2d) cudaStreamDestroy(P->h2d);
    if (P->d2h) cudaStreamDestroy(P->d2h);
    delete P;
    h->pipe = nullptr;
}

void matvec_host(svh_handle* h, const float2* I_host, float2* CC_host, int nrhs, bool green_only, int chunk,
                 cudaStream_t s) {
    const size_t per = (size_t)5 * h->K;
    const int cr = std::max(1, std::min(nrhs, chunk > 0 ? chunk : 4));
    if (!h->pipe || h->pipe->cap < (size_t)cr) {
        free_host_pipe(h);
        auto* P = new svh_handle::HostPipe();
        h->pipe = P;
        P->cap = cr;
        for (int k = 0; k < 2; ++k) {
            SVH_CUDA(cudaMalloc(&P->din[k], cr * per * sizeof(float2)));
            SVH_CUDA(cudaMalloc(&P->dout[k], cr * per * sizeof(float2)));
            SVH_CUDA(cudaEventCreateWithFlags(&P->in_ready[k], cudaEventDisableTiming));
            SVH_CUDA(cudaEventCreateWithFlags(&P->mv_done[k], cudaEventDisableTiming));
            SVH_CUDA(cudaEventCreateWithFlags(&P->out_done[k], cudaEventDisableTiming));
        }
        SVH_CUDA(cudaStreamCreateWithFlags(&P->h2d, cudaStreamNonBlocking));
        SVH_CUDA(cudaStreamCreateWithFlags(&P->d2h, cudaStreamNonBlocking));
    }
    auto* P = h->pipe;
    // order the pipeline after earlier work on the caller's stream
    SVH_CUDA(cudaEventRecord(P->mv_done[0], s));
    SVH_CUDA(cudaStreamWaitEvent(P->h2d, P->mv_done[0], 0));
    SVH_CUDA(cudaEventRecord(P->mv_done[1], s));
    const int nch = (nrhs + cr - 1) / cr;
    for (int c = 0; c < nch; ++c) {
        const int k = c & 1, r0 = c * cr, nr = std::min(cr, nrhs - r0);
        const size_t bytes = (size_t)nr * per * sizeof(float2);
        // slot k: its input was last read by the matvec of chunk c-2, its output by the D2H of c-2
        SVH_CUDA(cudaStreamWaitEvent(P->h2d, P->mv_done[k], 0));
        SVH_CUDA(cudaMemcpyAsync(P->din[k], I_host + r0 * per, bytes, cudaMemcpyHostToDevice, P->h2d));
        SVH_CUDA(cudaEventRecord(P->in_ready[k], P->h2d));
        SVH_CUDA(cudaStreamWaitEvent(s, P->in_ready[k], 0));
        if (c >= 2) SVH_CUDA(cudaStreamWaitEvent(s, P->out_done[k], 0));
        matvec(h, P->din[k], P->dout[k], nr, green_only, true, s);
        SVH_CUDA(cudaEventRecord(P->mv_done[k], s));
        SVH_CUDA(cudaStreamWaitEvent(P->d2h, P->mv_done[k], 0));
        SVH_CUDA(cudaMemcpyAsync(CC_host + r0 * per, P->dout[k], bytes, cudaMemcpyDeviceToHost, P->d2h));
        SVH_CUDA(cudaEventRecord(P->out_done[k], P->d2h));
    }
    for (int k = 0; k < 2 && k < nch; ++k) SVH_CUDA(cudaStreamWaitEvent(s, P->out_done[k], 0));
    SVH_CUDA(cudaStreamSynchronize(s));
}

}  // namespace svh
