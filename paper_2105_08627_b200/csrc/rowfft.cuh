// Row passes A and E of the matvec (Eq. 9) for row lengths 128 <= N <= 4096:
// a Stockham radix-16 FFT per row, 16 points per thread.
//
//   N = 16 x 16 x ... x R_last      (128 = 16*8, 256 = 16*16, 512 = 16*16*2,
//                                    1024 = 16*16*4, 2048 = 16*16*8, 4096 = 16*16*16)
//
// Stage s (radix R, Ns = 16^s) maps task t (k = t mod Ns) to
//   v[r] = src[t + r N/R] * W_{Ns R}^{k r},  v = FFT_R(v),  dst[(t/Ns) Ns R + k + r Ns] = v[r]
// (Stockham autosort: natural order in, natural order out).  The first stage reads the row
// straight from HBM (coalesced over t) and the last stage writes straight to HBM (its
// destination index is t + r N/R); only the middle exchanges go through shared memory,
// ping-pong buffers padded by one element per 16 (conflict-free for every stage's access
// pattern).  Zero padding (forward: inputs n >= N/2 are zero) prunes the first
// stage to R/2 loads and a half-input FFT; cropping (inverse: outputs n >= N/2 are never
// kept) prunes the last stage's stores.
//
// The twiddles W_{Ns R}^{k r} depend only on the thread, not on the row: the CTA walks
// many rows (persistent grid) and keeps the second stage's twiddles in registers.
#pragma once
#include "fft.cuh"

namespace svh {

template <int N>
struct RowPlan {
    static_assert(N >= 128 && N <= 4096 && (N & (N - 1)) == 0, "row plan: 128 <= N <= 4096, power of two");
    static constexpr int P = 16;                       // points per thread
    static constexpr int T = N / P;                    // threads per row
    static constexpr int RPC = T >= 128 ? 1 : 128 / T; // rows per CTA
    static constexpr int NT = T * RPC;                 // threads per CTA
    static constexpr int NS = N <= 256 ? 2 : 3;        // stages
    static constexpr int RL = N <= 256 ? N / 16 : N / 256;   // radix of the last stage
    static constexpr int PADN = N + N / 16;            // padded row length in shared memory
    static constexpr size_t smem = (size_t)RPC * 2 * PADN * sizeof(float2);   // B0 / B1 (slots follow)
    // blocks per SM targeted by the launch bounds (registers <= 65536 / (NT * MINB))
    static constexpr int MINB = NT >= 256 ? 2 : 4;
};

__device__ __forceinline__ int rpad(int i) { return i + (i >> 4); }

// W_N^e for e in [0, N): forward table value, conjugated for the inverse
template <int DIR>
__device__ __forceinline__ float2 tw_at(const float2* __restrict__ tw, int e) {
    float2 w = __ldg(&tw[e]);
    if (DIR > 0) w.y = -w.y;
    return w;
}

// one middle / last Stockham stage task of radix R at Ns for thread-local data v (already loaded)
template <int R, int DIR>
__device__ __forceinline__ void stage_twiddle(float2 (&v)[R], const float2 (&w)[R]) {
#pragma unroll
    for (int r = 1; r < R; ++r) v[r] = cmul(v[r], w[r]);
}

__device__ __forceinline__ void cpa8(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
                 "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void cpa16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
                 "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void cpa4(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
                 "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cpa_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
__device__ __forceinline__ void cpa_wait0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// Row segment of the packed order: the voxels of lattice row `row` are the packed indices
// [pre, pre + cnt) (x-fastest lexicographic order, P:45 / DESIGN.md §4).  rowinfo carries one
// sentinel row (index rows) whose first word holds K, so cnt = next row's pre - pre.
__device__ __forceinline__ int2 row_segment(const int2* __restrict__ rowinfo, int W, int row) {
    const int pre = __ldg(&rowinfo[(int64_t)row * W]).y;
    const int nxt = __ldg(&rowinfo[(int64_t)(row + 1) * W]).y;
    return make_int2(pre, nxt - pre);
}

// shared-memory slot of one row for the cp.async prefetch (double-buffered)
template <int N>
struct RowSlot {
    static constexpr int W = (N / 2 + 31) / 32;   // occupancy words of a row (Kx <= N/2)
    // RI [W] int2 | V [N/2] float2 (pass A: the row's packed inputs; pass E: its packed I)
    // | X [N] float2 (pass E only: the X1 row) | M [N/2 + 16] u8 (pass E only: material ids)
    static constexpr size_t A_b = (size_t)W * 8 + (size_t)(N / 2) * 8;
    static constexpr size_t E_b = A_b + (size_t)N * 8 + ((N / 2 + 16 + 15) / 16) * 16;
};

// Pass A: gather from packed order (or grid layout) + zero-pad + forward x-FFT, for the
// non-empty rows rowlist[0..nlist) of nrc = 5 nrhs (rhs, component) pairs.  X1 = [rc][rows][N].
// Each row's packed segment and occupancy words are copied HBM -> shared memory with cp.async
// one row-group ahead (the gather then runs on chip; no dependent HBM loads on the FFT path).
template <int N, bool PACKED>
__global__ void __launch_bounds__(RowPlan<N>::NT, RowPlan<N>::MINB)
    k_rowA(const float2* __restrict__ in, float2* __restrict__ X1, const int2* __restrict__ rowinfo, int W,
           const int32_t* __restrict__ rowlist, int nlist, const float2* __restrict__ tw, int Kx, int rows,
           int64_t K, int64_t Kt, int Ky, int Kyl, int y0, int nrc) {
    using PL = RowPlan<N>;
    using SL = RowSlot<N>;
    constexpr int T = PL::T, RPC = PL::RPC, PADN = PL::PADN, RL = PL::RL, NS = PL::NS;
    extern __shared__ __align__(16) unsigned char smraw[];
    const int q = threadIdx.x / T, j = threadIdx.x % T;
    float2* B0 = reinterpret_cast<float2*>(smraw) + q * 2 * PADN;
    float2* B1 = B0 + PADN;
    unsigned char* slots = smraw + PL::smem + (size_t)q * 2 * SL::A_b;
    const float2 zero = make_float2(0.f, 0.f);
    float2 w1[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) w1[r] = NS == 3 ? tw_at<-1>(tw, ((j & 15) * r * (N / 256)) & (N - 1)) : zero;
    const int groups = (nlist + RPC - 1) / RPC;
    const int total = groups * nrc;
    // bookkeeping loads (row list -> row-occupancy words) run two units ahead and are consumed
    // one iteration after issue: no dependent L2 latency on the critical path of a row
    auto row_load = [&](int u) -> int {
        if (u >= total) return -1;
        const int rc = u / groups;
        const int li = (u - rc * groups) * RPC + q;
        return li < nlist ? __ldg(&rowlist[li]) : -1;
    };
    auto seg_load = [&](int row, int& pre, int& nxt) {
        if (row < 0) {
            pre = nxt = 0;
        } else if (PACKED) {
            pre = __ldg(&rowinfo[(int64_t)row * W]).y;
            nxt = __ldg(&rowinfo[(int64_t)(row + 1) * W]).y;
        } else {
            pre = ((row / Ky) * Kyl + row % Ky - y0) * Kx;
            nxt = pre + Kx;
        }
    };
    // issue the copies of unit u (row `row`, packed segment [pre, pre + cnt)) into slot b
    auto issue = [&](int u, int row, int pre, int cnt, int b) {
        if (row >= 0) {
            const int rc = u / groups;
            unsigned char* sl = slots + b * SL::A_b;
            int2* RI = reinterpret_cast<int2*>(sl);
            float2* V = reinterpret_cast<float2*>(sl + SL::W * 8);
            if (PACKED)
                for (int e = j; e < W; e += T) cpa8(&RI[e], &rowinfo[(int64_t)row * W + e]);
            const float2* src = in + (PACKED ? (int64_t)rc * K : (int64_t)rc * Kt) + pre;
            for (int e = j; e < cnt; e += T) cpa8(&V[e], &src[e]);
        }
        cpa_commit();
    };
    const int G = gridDim.x;
    int u = blockIdx.x;
    int row0 = row_load(u), pre0, nxt0;
    seg_load(row0, pre0, nxt0);
    issue(u, row0, pre0, nxt0 - pre0, 0);
    int row1 = row_load(u + G), pre1, nxt1;
    seg_load(row1, pre1, nxt1);
    int row2 = row_load(u + 2 * G);
    for (int k = 0; u < total; ++k, u += G) {
        issue(u + G, row1, pre1, nxt1 - pre1, (k + 1) & 1);
        int pre2, nxt2;
        seg_load(row2, pre2, nxt2);
        const int row3 = row_load(u + 3 * G);
        const int row = row0;
        const int2 sg = make_int2(pre0, nxt0 - pre0);
        row0 = row1;
        pre0 = pre1;
        nxt0 = nxt1;
        row1 = row2;
        pre1 = pre2;
        nxt1 = nxt2;
        row2 = row3;
        const int rc = u / groups;
        cpa_wait1();
        __syncthreads();
        const int lrow = row >= 0 ? (row / Ky) * Kyl + row % Ky - y0 : 0;
        const unsigned char* sl = slots + (k & 1) * SL::A_b;
        const int2* RI = reinterpret_cast<const int2*>(sl);
        const float2* V = reinterpret_cast<const float2*>(sl + SL::W * 8);
        // stage 0: radix 16, Ns = 1, inputs n = j + r N/16 (r < 8 live: n < N/2)
        {
            float2 v[16];
#pragma unroll
            for (int r = 0; r < 16; ++r) v[r] = zero;
            if (row >= 0) {
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    const int n = j + r * (N / 16);
                    if (n < Kx) {
                        if (PACKED) {
                            const int2 mp = RI[n >> 5];
                            const unsigned bits = (unsigned)mp.x, b = (unsigned)(n & 31);
                            if ((bits >> b) & 1u) v[r] = V[mp.y - sg.x + __popc(bits & ((1u << b) - 1u))];
                        } else {
                            v[r] = V[n];
                        }
                    }
                }
            }
            reg_fft<16, -1, true>(v);
#pragma unroll
            for (int r = 0; r < 16; ++r) B0[rpad(j * 16 + r)] = v[r];
        }
        __syncthreads();
        float2* dst = X1 + ((int64_t)rc * rows + lrow) * N;
        if constexpr (NS == 2) {
            // last stage: radix RL = N/16, Ns = 16, tasks t = j + i T < 16 (16/RL per thread),
            // twiddle W_{16 RL}^{t r} = W_N^{t r}, destination t + 16 r
#pragma unroll
            for (int i = 0; i < 16 / RL; ++i) {
                const int t = j + i * T;
                float2 v[RL];
#pragma unroll
                for (int r = 0; r < RL; ++r) v[r] = B0[rpad(t + r * 16)];
#pragma unroll
                for (int r = 1; r < RL; ++r) v[r] = cmul(v[r], tw_at<-1>(tw, (t * r) & (N - 1)));
                reg_fft<RL, -1>(v);
                if (row >= 0) {
#pragma unroll
                    for (int r = 0; r < RL; ++r) dst[t + r * 16] = v[r];
                }
            }
        } else {
            // stage 1: radix 16, Ns = 16, task t = j (k = j mod 16)
            {
                float2 v[16];
#pragma unroll
                for (int r = 0; r < 16; ++r) v[r] = B0[rpad(j + r * (N / 16))];
                stage_twiddle<16, -1>(v, w1);
                reg_fft<16, -1>(v);
                const int base = (j >> 4) * 256 + (j & 15);
#pragma unroll
                for (int r = 0; r < 16; ++r) B1[rpad(base + r * 16)] = v[r];
            }
            __syncthreads();
            // stage 2 (last): radix RL, Ns = 256, tasks t = j + i T, k = t (t < N/RL = 256)
#pragma unroll
            for (int i = 0; i < 16 / RL; ++i) {
                const int t = j + i * T;
                float2 v[RL];
#pragma unroll
                for (int r = 0; r < RL; ++r) v[r] = B1[rpad(t + r * (N / RL))];
#pragma unroll
                for (int r = 1; r < RL; ++r) v[r] = cmul(v[r], tw_at<-1>(tw, (t * r) & (N - 1)));
                reg_fft<RL, -1>(v);
                if (row >= 0) {
#pragma unroll
                    for (int r = 0; r < RL; ++r) dst[t + r * (N / RL)] = v[r];
                }
            }
        }
        // NS == 2: B0 is rewritten by the next unit's stage 0 -- its barrier after the copy wait
        // orders that write after every thread's reads here (each thread passes it only after
        // finishing this iteration)
    }
    cpa_wait0();
}

// Pass E: inverse x-FFT + crop + local term z^b I^b + scatter to packed order (or
// grid layout), over the rows rowlist[li] (packed output: the non-empty rows) or every row of
// the (slab) grid (rowlist == nullptr, grid output: empty rows are written as zeros).  The
// row's occupancy words, packed I segment and material ids are copied to shared memory with
// cp.async one row-group ahead, the X1 row as soon as the previous one has been read; the
// packed outputs are assembled in place of the I segment and leave as one contiguous,
// coalesced segment.  One FFT buffer (in place, one extra barrier) keeps a 2048-point row
// group at ~52 KB of shared memory: four CTAs per SM.
template <int N>
struct RowSlotE {
    static constexpr int W = (N / 2 + 31) / 32;
    // small slot (double-buffered): RI [W] int2 | V [N/2] float2 | M [N/2 + 16] u8
    static constexpr size_t S_b = (size_t)W * 8 + (size_t)(N / 2) * 8 + ((N / 2 + 16 + 15) / 16) * 16;
    // per row group: B [PADN] float2 | X [N] float2 | 2 small slots
    static constexpr size_t G_b = (size_t)RowPlan<N>::PADN * 8 + (size_t)N * 8 + 2 * S_b;
};

template <int N, bool PACKED>
__global__ void __launch_bounds__(RowPlan<N>::NT, RowPlan<N>::MINB)
    k_rowE(const float2* __restrict__ X1, float2* __restrict__ out, const float2* __restrict__ in,
           const int2* __restrict__ rowinfo, int W, const int32_t* __restrict__ rowlist, int nlist,
           const uint32_t* __restrict__ rowmask, int rowMW, int Ky, const uint8_t* __restrict__ matp,
           const float2* __restrict__ zloc, int nzl, const float2* __restrict__ tw, int Kx, int rows, int64_t K,
           int64_t Kt, int green_only, int Kyl, int y0, int nrc) {
    using PL = RowPlan<N>;
    using SL = RowSlotE<N>;
    constexpr int T = PL::T, RPC = PL::RPC, PADN = PL::PADN, RL = PL::RL, NS = PL::NS;
    extern __shared__ __align__(16) unsigned char smraw[];
    const int q = threadIdx.x / T, j = threadIdx.x % T;
    unsigned char* grp = smraw + (size_t)q * SL::G_b;
    float2* B = reinterpret_cast<float2*>(grp);
    float2* X = reinterpret_cast<float2*>(grp + (size_t)PADN * 8);
    unsigned char* slots = grp + (size_t)PADN * 8 + (size_t)N * 8;
    const float2 zero = make_float2(0.f, 0.f);
    float2 w1[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) w1[r] = NS == 3 ? tw_at<+1>(tw, ((j & 15) * r * (N / 256)) & (N - 1)) : zero;
    const int groups = (nlist + RPC - 1) / RPC;
    const int total = groups * nrc;
    // bookkeeping loads (row list -> row-occupancy words / row mask) run two units ahead and
    // are consumed one iteration after issue (no dependent L2 latency on a row's critical path)
    auto row_load = [&](int u) -> int {
        if (u >= total) return -1;
        const int rc = u / groups;
        const int li = (u - rc * groups) * RPC + q;
        if (li >= nlist) return -1;
        return rowlist ? __ldg(&rowlist[li]) : (li / Kyl) * Ky + y0 + li % Kyl;
    };
    auto seg_load = [&](int row, int& pre, int& nxt, uint32_t& lw) {
        lw = 0;
        if (row < 0) {
            pre = nxt = 0;
            return;
        }
        if (PACKED) {
            pre = __ldg(&rowinfo[(int64_t)row * W]).y;
            nxt = __ldg(&rowinfo[(int64_t)(row + 1) * W]).y;
        } else {
            pre = ((row / Ky) * Kyl + row % Ky - y0) * Kx;
            nxt = pre + Kx;
        }
        lw = rowlist ? 1u : (__ldg(&rowmask[(int64_t)(row / Ky) * rowMW + ((row % Ky) >> 5)]) >> ((row % Ky) & 31));
    };
    auto issue_small = [&](int u, int row, int2 sg, bool live, int b) {
        if (row >= 0) {
            const int rc = u / groups;
            unsigned char* sl = slots + b * SL::S_b;
            int2* RI = reinterpret_cast<int2*>(sl);
            float2* V = reinterpret_cast<float2*>(sl + SL::W * 8);
            uint32_t* Mw = reinterpret_cast<uint32_t*>(sl + SL::W * 8 + (N / 2) * 8);
            for (int e = j; e < W; e += T) cpa8(&RI[e], &rowinfo[(int64_t)row * W + e]);
            if (!green_only && live) {
                const float2* src = in + (PACKED ? (int64_t)rc * K : (int64_t)rc * Kt) + sg.x;
                for (int e = j; e < sg.y; e += T) cpa8(&V[e], &src[e]);
                if (PACKED) {   // material ids of the segment, 4-byte words (matp is padded)
                    const int a0 = sg.x & ~3, nw = (sg.x + sg.y - a0 + 3) >> 2;
                    for (int e = j; e < nw; e += T) cpa4(&Mw[e], matp + a0 + 4 * e);
                }
            }
        }
        cpa_commit();
    };
    auto issue_x = [&](int u, int row, bool live) {
        if (live) {
            const int rc = u / groups;
            const int lrow = (row / Ky) * Kyl + row % Ky - y0;
            const float2* xr = X1 + ((int64_t)rc * rows + lrow) * N;
            for (int e = j; e < N / 2; e += T) cpa16(&X[2 * e], &xr[2 * e]);
        }
        cpa_commit();
    };
    const int G = gridDim.x;
    int u = blockIdx.x;
    int row0 = row_load(u), pre0, nxt0;
    uint32_t lw0;
    seg_load(row0, pre0, nxt0, lw0);
    issue_small(u, row0, make_int2(pre0, nxt0 - pre0), (lw0 & 1u) != 0, 0);
    issue_x(u, row0, row0 >= 0 && (lw0 & 1u));
    int row1 = row_load(u + G), pre1, nxt1;
    uint32_t lw1;
    seg_load(row1, pre1, nxt1, lw1);
    int row2 = row_load(u + 2 * G);
    for (int k = 0; u < total; ++k, u += G) {
        cpa_wait0();
        __syncthreads();   // this row's copies landed; every thread is done with the previous row
        const bool live1 = row1 >= 0 && (lw1 & 1u);
        issue_small(u + G, row1, make_int2(pre1, nxt1 - pre1), live1, (k + 1) & 1);
        int pre2, nxt2;
        uint32_t lw2;
        seg_load(row2, pre2, nxt2, lw2);
        const int row3 = row_load(u + 3 * G);
        const int row = row0;
        const int2 sg = make_int2(pre0, nxt0 - pre0);
        const bool live = row0 >= 0 && (lw0 & 1u);
        const int rc = u / groups;
        const int comp = rc % 5;
        unsigned char* sl = slots + (k & 1) * SL::S_b;
        const int2* RI = reinterpret_cast<const int2*>(sl);
        float2* V = reinterpret_cast<float2*>(sl + SL::W * 8);
        const uint8_t* Mb = sl + SL::W * 8 + (N / 2) * 8 + (sg.x & 3);
        // output element n (< Kx): local term, into the segment staging in place of I (each
        // position is read and written by one thread)
        auto put = [&](int n, float2 v) {
            if (row < 0 || n >= Kx) return;
            const int2 mp = RI[n >> 5];
            const unsigned bits = (unsigned)mp.x, b = (unsigned)(n & 31);
            if (PACKED) {
                if (!((bits >> b) & 1u)) return;
                const int o = mp.y - sg.x + __popc(bits & ((1u << b) - 1u));
                if (!green_only) v = cadd(v, cmul(__ldg(&zloc[Mb[o] * 5 + comp]), V[o]));
                V[o] = v;
            } else {
                if (!((bits >> b) & 1u)) {
                    V[n] = zero;
                    return;
                }
                if (!green_only) {
                    const int idx = mp.y + __popc(bits & ((1u << b) - 1u));
                    v = cadd(v, cmul(__ldg(&zloc[__ldg(&matp[idx]) * 5 + comp]), V[n]));
                }
                V[n] = v;
            }
        };
        // stage 0: radix 16, Ns = 1, all N inputs (from the X copy)
        {
            float2 v[16];
#pragma unroll
            for (int r = 0; r < 16; ++r) v[r] = live ? X[j + r * (N / 16)] : zero;
            reg_fft<16, +1>(v);
#pragma unroll
            for (int r = 0; r < 16; ++r) B[rpad(j * 16 + r)] = v[r];
        }
        __syncthreads();
        issue_x(u + G, row1, live1);   // X is free: the next row's X1 row streams in meanwhile
        if constexpr (NS == 2) {
#pragma unroll
            for (int i = 0; i < 16 / RL; ++i) {
                const int t = j + i * T;
                float2 v[RL];
#pragma unroll
                for (int r = 0; r < RL; ++r) v[r] = B[rpad(t + r * 16)];
#pragma unroll
                for (int r = 1; r < RL; ++r) v[r] = cmul(v[r], tw_at<+1>(tw, (t * r) & (N - 1)));
                reg_fft<RL, +1>(v);
#pragma unroll
                for (int r = 0; r < RL / 2; ++r) put(t + r * 16, v[r]);
            }
        } else {
            {
                float2 v[16];
#pragma unroll
                for (int r = 0; r < 16; ++r) v[r] = B[rpad(j + r * (N / 16))];
                __syncthreads();   // in place: every stage-1 read before any stage-1 write
                stage_twiddle<16, +1>(v, w1);
                reg_fft<16, +1>(v);
                const int base = (j >> 4) * 256 + (j & 15);
#pragma unroll
                for (int r = 0; r < 16; ++r) B[rpad(base + r * 16)] = v[r];
            }
            __syncthreads();
#pragma unroll
            for (int i = 0; i < 16 / RL; ++i) {
                const int t = j + i * T;
                float2 v[RL];
#pragma unroll
                for (int r = 0; r < RL; ++r) v[r] = B[rpad(t + r * (N / RL))];
#pragma unroll
                for (int r = 1; r < RL; ++r) v[r] = cmul(v[r], tw_at<+1>(tw, (t * r) & (N - 1)));
                reg_fft<RL, +1>(v);
#pragma unroll
                for (int r = 0; r < RL / 2; ++r) put(t + r * (N / RL), v[r]);
            }
        }
        __syncthreads();   // the staged segment is complete
        if (row >= 0) {
            float2* dst = out + (PACKED ? (int64_t)rc * K : (int64_t)rc * Kt) + sg.x;
            for (int e = j; e < sg.y; e += T) dst[e] = V[e];
        }
        row0 = row1;
        pre0 = pre1;
        nxt0 = nxt1;
        lw0 = lw1;
        row1 = row2;
        pre1 = pre2;
        nxt1 = nxt2;
        lw1 = lw2;
        row2 = row3;
    }
    cpa_wait0();
}

}  // namespace svh
