// Pass C of the matvec (Eq. 9; Tucker restoration P:89-101) on the BLOCKED X2 layout
// of the 2048-point y passes:  X2 = [rc][ky][kx / 8][z][kx % 8]  (ypass.cuh, kZB = 8).
//
// In the plane-major layout [rc][z][ky][kx] a z pencil is strided by a whole plane, so pass C
// moved 128-byte pieces at 32 MB strides (k_zpass: DRAM 28 % of peak, 10 warps per SM behind
// CTA barriers).  In the blocked layout the 5 x Kz x 8 points of one (RHS, ky, kx block) tile
// are five CONTIGUOUS chunks of 8 Kz points: each moves with one 1-D bulk copy (TMA,
// cp.async.bulk) into a 2-deep mbarrier ring, and leaves by five bulk stores from the same
// slot.  The tile is small (Q = 8 pencils per component), so two CTAs share an SM.
//
// Work unit = (oy, kx block): the rows ky = oy and Ny - oy share their raw kernel spectra (K1y
// flips sign), built once per unit (Tucker expansion on chip, or the dense octant) and used for
// both rows and every RHS.  The z-FFT is split N = R1 x R2 as in zpass.cuh:
//   L1 (thread (c, n2, q)):  R1-point FFT over n1 of x[R2 n1 + n2] (the zero half pruned),
//                            read from the staged tile, written to the exchange buffer T;
//   L2 (thread (k1, q)):     twiddle, R2-point FFT of the 5 components, moment-form MAC,
//                            inverse R2-point FFT, inverse twiddle, back to T;
//   L1 inverse:              R1-point inverse FFT -> z = R2 n1 + n2 < Kz, into the staged tile,
//                            which then leaves by bulk stores.
#include <algorithm>
#include <cuda_runtime.h>

#include "fft.cuh"
#include "internal.h"
#include "tma.cuh"
#include "zpass.cuh"   // SpecView, kTuckerMaxRank

namespace svh {
namespace {

constexpr int kQB = 8;   // = kZB of ypass.cuh (kx per block of the blocked layout)

template <int N, int R2_, int NT_, int DM_>
struct ZBPlan {
    static constexpr int Q = kQB, R2 = R2_, R1 = N / R2_, NK = N / 2 + 1, NT = NT_, DM = DM_, DP = DM_ + 1;
    static constexpr int NL1 = 5 * R2 * Q, NL2 = R1 * Q;
    static constexpr int TL1 = NL1 / NT;
    static_assert(NL1 % NT == 0 && NL2 <= NT && NT % 32 == 0, "zblk plan: balanced L1, one L2 task per thread");
    static constexpr int S = 2;                                  // ring depth
    static constexpr int SE = 5 * (N / 2) * Q;                   // stage elements (Kz <= N/2)
    static constexpr int TB = R1 * Q + Q;                        // one (c, n2) block of T, padded
    static constexpr int TE = 5 * R2 * TB;
    static constexpr size_t stage_b = (size_t)S * SE * sizeof(float2);
    static constexpr size_t T_b = (size_t)TE * sizeof(float2);
    static constexpr size_t KV_b = (size_t)7 * NK * Q * sizeof(float);
    static constexpr size_t GH_b = DM ? ((size_t)7 * DM * DP + (size_t)7 * Q * DP) * sizeof(float) : 0;
    static constexpr size_t smem = stage_b + T_b + KV_b + GH_b + S * sizeof(uint64_t);
};

template <int N, int R2, int NT, int DM>
__global__ void __launch_bounds__(NT)
    k_zblk(float2* __restrict__ X2, SpecView sv, const float2* __restrict__ tw, int Nx, int Ny, int Kz, float g,
           int nrhs, const uint8_t* __restrict__ planeok) {
    using P = ZBPlan<N, R2, NT, DM>;
    constexpr int Q = P::Q, R1 = P::R1, NK = P::NK, TB = P::TB, TL1 = P::TL1, NL2 = P::NL2, S = P::S, SE = P::SE;
    constexpr int DP = P::DP;
    extern __shared__ __align__(128) unsigned char smraw[];
    float2* stage = reinterpret_cast<float2*>(smraw);                             // [S][5][Kz][Q]
    float2* T = reinterpret_cast<float2*>(smraw + P::stage_b);                    // [5][R2][TB]
    float* KV = reinterpret_cast<float*>(smraw + P::stage_b + P::T_b);           // [7][NK][Q]
    float* G = KV + 7 * NK * Q;                                                   // [7][DM][DP]
    float* H = G + 7 * DM * DP;                                                   // [7][Q][DP]
    uint64_t* bar = reinterpret_cast<uint64_t*>(smraw + P::stage_b + P::T_b + P::KV_b + P::GH_b);
    const int tid = threadIdx.x;
    const float2 zero = make_float2(0.f, 0.f);
    const int NB = Nx / Q;
    const int nunits = (Ny / 2 + 1) * NB;
    const int u0 = (int)((int64_t)nunits * blockIdx.x / gridDim.x);
    const int u1 = (int)((int64_t)nunits * (blockIdx.x + 1) / gridDim.x);
    const int64_t chunk = (int64_t)Kz * Q;                                        // points per chunk
    const uint32_t chunk_b = (uint32_t)(chunk * sizeof(float2));
    // L1 tasks a = tid + k NT -> (c, n2, q) and their live-input masks (planes holding voxels)
    int tc[TL1], tq[TL1], tn2[TL1];
    uint32_t live[TL1];
#pragma unroll
    for (int k = 0; k < TL1; ++k) {
        const int a = tid + k * NT;
        tc[k] = a / (R2 * Q);
        tn2[k] = (a / Q) % R2;
        tq[k] = a % Q;
        uint32_t m = 0;
        for (int n1 = 0; n1 < R1 / 2; ++n1) {
            const int z = R2 * n1 + tn2[k];
            if (z < Kz && __ldg(&planeok[z])) m |= 1u << n1;
        }
        live[k] = m;
    }
    const bool l2 = tid < NL2;
    const int k1 = tid / Q, q2 = tid % Q;
    float2 w2[R2];
#pragma unroll
    for (int m = 0; m < R2; ++m) w2[m] = l2 ? __ldg(&tw[(m * k1) & (N - 1)]) : zero;
    auto rows_of = [&](int u) { const int oy = u / NB; return (oy == 0 || 2 * oy == Ny) ? 1 : 2; };
    // tile (u, i): i = row * nrhs + r; chunk of component c at X2 + base + c * Ny * NB * chunk
    auto tile_base = [&](int u, int i, int& ky, int& kb) -> int64_t {
        const int oy = u / NB;
        kb = u % NB;
        const int row = i / nrhs, r = i % nrhs;
        ky = row == 0 ? oy : Ny - oy;
        return (((int64_t)r * 5 * Ny + ky) * NB + kb) * chunk;
    };
    const int64_t cstride = (int64_t)Ny * NB * chunk;                             // next component
    auto issue = [&](int u, int i, int st) {                                      // thread 0
        if (u >= u1) return;
        int ky, kb;
        const int64_t base = tile_base(u, i, ky, kb);
        mbar_arrive_expect_tx(&bar[st], 5 * chunk_b);
#pragma unroll
        for (int c = 0; c < 5; ++c) bulk_load(stage + st * SE + c * chunk, X2 + base + c * cstride, chunk_b, &bar[st]);
    };
    auto advance = [&](int& u, int& i) {
        if (++i == rows_of(u) * nrhs) {
            ++u;
            i = 0;
        }
    };
    if (tid == 0) {
        for (int st = 0; st < S; ++st) mbar_init(&bar[st], 1);
        mbar_fence_init();
    }
    __syncthreads();
    int iu = u0, ii = 0;   // issue cursor (S tiles ahead)
    if (tid == 0)
        for (int st = 0; st < S && iu < u1; ++st) {
            issue(iu, ii, st);
            advance(iu, ii);
        }
    if (tid != 0)
        for (int st = 0; st < S && iu < u1; ++st) advance(iu, ii);
    int cur_oy = -1;
    int u = u0, i = 0;
    for (int idx = 0; u < u1; ++idx) {
        const int st = idx % S;
        int ky, kb;
        const int64_t base = tile_base(u, i, ky, kb);
        const int oy = u / NB;
        if (i == 0) {
            // the unit's kernel values KV[m][kh][q] (the previous tile's L2 reads ended at its barrier)
            if constexpr (DM > 0) {
                if (oy != cur_oy) {
                    // G_m = core_m x2 F2_m[oy]  ([c3][c1], zero outside the ranks)
                    for (int t = tid; t < 7 * DM * DM; t += NT) {
                        const int m = t / (DM * DM), rest = t - m * DM * DM, c3 = rest / DM, c1 = rest - c3 * DM;
                        const int d1 = sv.rk[m][0], d2 = sv.rk[m][1], d3 = sv.rk[m][2];
                        float acc = 0.f;
                        if (c3 < d3 && c1 < d1) {
                            const float* cp = sv.core[m] + (int64_t)c3 * d2 * d1 + c1;
                            const float* F2 = sv.fac[m][1] + (int64_t)oy * d2;
                            for (int cc2 = 0; cc2 < d2; ++cc2) acc = fmaf(__ldg(&cp[cc2 * d1]), __ldg(&F2[cc2]), acc);
                        }
                        G[(m * DM + c3) * DP + c1] = acc;
                    }
                    cur_oy = oy;
                }
                __syncthreads();
                // H_m[q] = G_m x1 F1_m[ox_q]
                for (int t = tid; t < 7 * Q * DM; t += NT) {
                    const int m = t / (Q * DM), rest = t - m * Q * DM, q = rest / DM, c3 = rest - q * DM;
                    const int d1 = sv.rk[m][0];
                    const int kx = kb * Q + q;
                    const int ox = kx <= (Nx >> 1) ? kx : Nx - kx;
                    const float* f1 = sv.fac[m][0] + (int64_t)ox * d1;
                    const float* gr = G + (m * DM + c3) * DP;
                    float acc = 0.f;
                    for (int c = 0; c < d1; ++c) acc = fmaf(gr[c], __ldg(&f1[c]), acc);
                    H[(m * Q + q) * DP + c3] = acc;
                }
                __syncthreads();
                // KV[m][kh][q] = F3_m[kh] . H_m[q]
                for (int t = tid; t < 7 * NK * Q; t += NT) {
                    const int q = t % Q, rest = t / Q, kh = rest % NK, m = rest / NK;
                    const int d3 = sv.rk[m][2];
                    const float* f3 = sv.fac[m][2] + (int64_t)kh * d3;
                    const float* hq = H + (m * Q + q) * DP;
                    float acc = 0.f;
                    for (int c = 0; c < d3; ++c) acc = fmaf(__ldg(&f3[c]), hq[c], acc);
                    KV[t] = acc;
                }
            } else {
                const int64_t pl = (int64_t)sv.hx * sv.hy * sv.hz;
                for (int t = tid; t < 7 * NK * Q; t += NT) {
                    const int q = t % Q, rest = t / Q, kh = rest % NK, m = rest / NK;
                    const int kx = kb * Q + q;
                    const int ox = kx <= (Nx >> 1) ? kx : Nx - kx;
                    KV[t] = __ldg(&sv.spec[m * pl + ((int64_t)kh * sv.hy + oy) * sv.hx + ox]);
                }
            }
        }
        mbar_wait(&bar[st], (uint32_t)((idx / S) & 1));
        float2* sg = stage + st * SE;
        // L1 forward: staged inputs -> T
#pragma unroll
        for (int k = 0; k < TL1; ++k) {
            float2 v[R1];
            const float2* src = sg + tc[k] * chunk + tn2[k] * Q + tq[k];
#pragma unroll
            for (int n1 = 0; n1 < R1; ++n1) v[n1] = (n1 < R1 / 2 && ((live[k] >> n1) & 1u)) ? src[n1 * R2 * Q] : zero;
            reg_fft<R1, -1, true>(v);
            float2* t1 = T + (tc[k] * R2 + tn2[k]) * TB + tq[k];
#pragma unroll
            for (int kk = 0; kk < R1; ++kk) t1[kk * Q] = v[kk];
        }
        __syncthreads();   // T complete; KV built
        if (l2) {
            const int kx = kb * Q + q2;
            const float gx = kx <= (Nx >> 1) ? g : -g, gy = ky <= (Ny >> 1) ? g : -g;
            float2 uu[5][R2];
#pragma unroll
            for (int c = 0; c < 5; ++c) {
#pragma unroll
                for (int m = 0; m < R2; ++m) {
                    const float2 x = T[(c * R2 + m) * TB + k1 * Q + q2];
                    uu[c][m] = m ? cmul(x, w2[m]) : x;
                }
                reg_fft<R2, -1>(uu[c]);
            }
#pragma unroll
            for (int k2 = 0; k2 < R2; ++k2) {
                const int kz = k1 + R1 * k2;
                const int kh = kz <= (N >> 1) ? kz : N - kz;
                const float s3 = kz <= (N >> 1) ? 1.f : -1.f;   // K1z is odd in kz
                const float* kv = KV + kh * Q + q2;
                const float f0 = g * kv[0 * NK * Q], f1 = gx * kv[1 * NK * Q], f2 = gy * kv[2 * NK * Q];
                const float f3 = (-2.f * g) * s3 * kv[3 * NK * Q];
                const float f4 = g * kv[4 * NK * Q], f5 = g * kv[5 * NK * Q], f6 = (4.f * g) * kv[6 * NK * Q];
                const float2 Ix = uu[0][k2], Iy = uu[1][k2], Iz = uu[2][k2], I2 = uu[3][k2], I3 = uu[4][k2];
                const float2 m1x = cadd(I2, I3), m1y = csub(I3, I2);
                const float2 Qx = cfma_s(Ix, -f1, cmul_i(m1x, f4));
                const float2 Qy = cfma_s(Iy, -f2, cmul_i(m1y, f5));
                const float2 Qz = cfma_s(Iz, -f3, cmul_i(I3, f6));
                uu[0][k2] = cfma_s(m1x, f1, cmul_i(Ix, f0));
                uu[1][k2] = cfma_s(m1y, f2, cmul_i(Iy, f0));
                uu[2][k2] = cfma_s(I3, f3, cmul_i(Iz, f0));
                uu[3][k2] = csub(Qx, Qy);
                uu[4][k2] = cadd(cadd(Qx, Qy), Qz);
            }
#pragma unroll
            for (int c = 0; c < 5; ++c) {
                reg_fft<R2, +1>(uu[c]);
#pragma unroll
                for (int m = 0; m < R2; ++m) {
                    const float2 wc = make_float2(w2[m].x, -w2[m].y);
                    T[(c * R2 + m) * TB + k1 * Q + q2] = m ? cmul(uu[c][m], wc) : uu[c][m];
                }
            }
        }
        __syncthreads();
        // L1 inverse: z = n2 + R2 n1 < Kz back into the staged tile
#pragma unroll
        for (int k = 0; k < TL1; ++k) {
            float2 v[R1];
            const float2* t1 = T + (tc[k] * R2 + tn2[k]) * TB + tq[k];
#pragma unroll
            for (int kk = 0; kk < R1; ++kk) v[kk] = t1[kk * Q];
            reg_fft<R1, +1>(v);
            float2* dst = sg + tc[k] * chunk + tn2[k] * Q + tq[k];
#pragma unroll
            for (int n1 = 0; n1 < R1 / 2; ++n1)
                if (R2 * n1 + tn2[k] < Kz) dst[n1 * R2 * Q] = v[n1];
        }
        fence_proxy_async_smem();
        __syncthreads();   // tile written back; T free for the next tile
        if (tid == 0) {
#pragma unroll
            for (int c = 0; c < 5; ++c) bulk_store(X2 + base + c * cstride, sg + c * chunk, chunk_b);
            tma_store_commit();
            bulk_wait_read<0>();   // the slot is re-filled next: its stores must have read it
            issue(iu, ii, st);
        }
        if (iu < u1) advance(iu, ii);
        advance(u, i);
    }
    if (tid == 0) tma_store_wait0();
}

template <int N, int R2, int NT, int DM>
void launch(svh_handle* h, float2* X2, int nrhs, const SpecView& sv, cudaStream_t s) {
    using P = ZBPlan<N, R2, NT, DM>;
    auto kern = k_zblk<N, R2, NT, DM>;
    static thread_local int ctas[64] = {};   // per device: attributes set + resident CTAs (once)
    int dev = 0;
    cudaGetDevice(&dev);
    if (ctas[dev & 63] == 0) {
        SVH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                      (int)cudaSharedmemCarveoutMaxShared));
        SVH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P::smem));
        int nsm = 148, occ = 1;
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, P::smem);
        ctas[dev & 63] = nsm * std::max(occ, 1);
    }
    const int64_t units = (int64_t)(h->ny / 2 + 1) * (h->nx / kQB);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(units, ctas[dev & 63]));
    SVH_LAUNCH(kern, grid, NT, P::smem, s, X2, sv, h->d_tw[2], h->nx, h->ny, h->kz, h->gscale, nrhs, h->d_planeok);
}

}  // namespace

int zblk_max_rank(const svh_handle* h) {
    int d = 0;
    if (h->use_tucker)
        for (int m = 0; m < 7; ++m)
            for (int a = 0; a < 3; ++a) d = std::max(d, h->tucker.ranks[m][a]);
    return d;
}

// the blocked X2 layout is used iff the whole-grid y passes are the 2048-point k_ypass and this
// pass C handles the z extent
bool zblk_supported(const svh_handle* h) {
    return h->ny == 2048 && (h->nz == 64 || h->nz == 128) && h->nx % kQB == 0 &&
           zblk_max_rank(h) <= kTuckerMaxRank;
}

void run_zblk(svh_handle* h, float2* X2, int nrhs, cudaStream_t s) {
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
    const int dm = zblk_max_rank(h);
    auto go = [&](auto Nc, auto R2c) {
        constexpr int N = decltype(Nc)::value, R2 = decltype(R2c)::value;
        constexpr int NT = 5 * R2 * kQB / 2;   // two L1 tasks per thread (160)
        if (!h->use_tucker)
            launch<N, R2, NT, 0>(h, X2, nrhs, sv, s);
        else if (dm <= 16)
            launch<N, R2, NT, 16>(h, X2, nrhs, sv, s);
        else
            launch<N, R2, NT, 32>(h, X2, nrhs, sv, s);
    };
    if (h->nz == 64)
        go(std::integral_constant<int, 64>{}, std::integral_constant<int, 8>{});
    else
        go(std::integral_constant<int, 128>{}, std::integral_constant<int, 8>{});
}

}  // namespace svh
