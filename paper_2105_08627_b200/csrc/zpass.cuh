// Pass C of the matvec for 64 <= Nz <= 256 (Eq. 9; Tucker restoration P:89-101):
// z-FFT of the 5 embedded current components, the 5 -> 5 moment-form MAC with the 7 kernel
// spectra, inverse z-FFT and crop, in place on X2 = [rc][Kz][Ny][Nxs].
//
// Work unit = (oy, kx tile of Q columns): the rows ky = oy and Ny - oy share their raw kernel
// spectra (K1y only flips sign, applied in the MAC), so the 7 x (N/2 + 1) x Q raw values are
// built once per unit -- by the on-chip Tucker expansion (Eq. 10) or from the dense octant --
// and used for both rows and every right-hand side.  A tile = one (RHS, row, kx tile).
//
// The z-FFT is split N = R1 x R2 (R1 = 16/32, R2 = 4/8):
//   L1 (thread (c, n2, q)):  R1-point FFT over n1 of x[R2 n1 + n2] (inputs z >= N/2 are the zero
//                            padding: R1/2 loads, straight from HBM into registers, prefetched one
//                            tile ahead), written to the exchange buffer T;
//   L2 (thread (k1, q)):     all 5 components: twiddle W_N^{n2 k1}, R2-point FFT -> kz = k1 + R1 k2,
//                            MAC in registers, inverse R2-point FFT, twiddle W_N^{-n2 k1}, back to T;
//   L1 inverse:              R1-point inverse FFT over k1 -> z = n2 + R2 n1, the kept z < Kz are
//                            stored straight to HBM.
// L1 needs no twiddles (compile-time constants); L2's R2-1 twiddles are per-thread constants.
// Two barriers per tile: a thread's forward L1 of the next tile rewrites only the T pencils its own
// inverse L1 has just read, so one T buffer needs no third barrier.
#pragma once
#include "fft.cuh"
#include "tma.cuh"

namespace svh {

// largest Tucker rank the on-chip expansion handles (ranks of the 7 kernels, SURVEY 8(c) P15:
// 10-21 for tol 1e-4 .. 1e-10); higher ranks take the generic z pass (k_freq_big)
constexpr int kTuckerMaxRank = 32;

struct SpecView {
    const float* spec;   // dense [7][hz][hy][hx]; null in Tucker mode
    int hx, hy, hz;
    // Tucker mode (Eq. 10): factors [7][3] -> fp32 [h_i][d_i], cores [7] -> fp32 [d3][d2][d1]
    const float* fac[7][3];
    const float* core[7];
    int rk[7][3];
};

template <int N, int R2_, int Q_, int NT_>
struct ZPlan {
    static constexpr int R2 = R2_, Q = Q_, R1 = N / R2_, NH = N / 2, NK = N / 2 + 1;
    static constexpr int NL1 = 5 * R2 * Q, NL2 = R1 * Q;
    static constexpr int NT = NT_;
    static constexpr int TL1 = NL1 / NT;                  // L1 tasks per thread
    static_assert(NL1 % NT == 0 && NL2 <= NT && NT % 32 == 0, "z plan: balanced L1, one L2 task per thread");
    static constexpr int TB = R1 * Q + Q;                 // one (c, n2) block of T, padded by Q
    static constexpr int TE = 5 * R2 * TB;                // elements of one T buffer
    static constexpr int KVS = 8;                         // floats per (kh, q) entry of KV (7 used)
    static constexpr size_t KV_b = (size_t)NK * Q * KVS * sizeof(float);
    // T (double-buffered in dense mode) | KV [NK][Q][8] | Tucker (rank bucket DM > 0): the
    // mode-3 factor rows F3 [7][NK][DM], G [7][DM][DM + 1], H [7][Q][DM + 1] (zero-padded to DM)
    static constexpr size_t smem(int nbuf, int DM) {
        return (size_t)nbuf * TE * sizeof(float2) + KV_b +
               (DM ? ((size_t)7 * NK * DM + (size_t)7 * DM * (DM + 1) + (size_t)7 * Q * (DM + 1)) * sizeof(float) : 0);
    }
};

// NBUF = 2: T double-buffered; 1: single buffer (two barriers per tile either way).
// DM = 0: dense octant spectra; 16 / 32: Tucker factors, ranks <= DM (zero-padded on chip).
template <int N, int R2, int Q, int NT, int NBUF, int DM>
__global__ void __launch_bounds__(NT, 1)
    k_zpass(float2* __restrict__ X2, SpecView sv, const float2* __restrict__ tw, int Nx, int Ny, int Kz, int Nxs,
            int kxg, float g, int nrhs, const uint8_t* __restrict__ planeok) {
    using P = ZPlan<N, R2, Q, NT>;
    constexpr int R1 = P::R1, NK = P::NK, TB = P::TB, TE = P::TE, TL1 = P::TL1, NL2 = P::NL2, KVS = P::KVS;
    constexpr int DP = DM + 1;   // padded row of G / H (conflict-free column reads)
    extern __shared__ __align__(16) unsigned char smraw[];
    float2* T = reinterpret_cast<float2*>(smraw);                                 // [NBUF][5][R2][TB]
    float* KV = reinterpret_cast<float*>(smraw + (size_t)NBUF * TE * sizeof(float2));   // [NK][Q][8]
    float* F3s = KV + NK * Q * KVS;                                               // [7][NK][DM]
    float* G = F3s + 7 * NK * DM;                                                 // [7][DM][DP]
    float* H = G + 7 * DM * DP;                                                   // [7][Q][DP]
    const int tid = threadIdx.x;
    const float2 zero = make_float2(0.f, 0.f);
    const int64_t plane = (int64_t)Nxs * Ny;
    const int tiles_x = Nxs / Q;
    const int nunits = (Ny / 2 + 1) * tiles_x;
    const int u0 = (int)((int64_t)nunits * blockIdx.x / gridDim.x);
    const int u1 = (int)((int64_t)nunits * (blockIdx.x + 1) / gridDim.x);
    // L1 tasks a = tid + k NT -> (c, n2, q); their element pointers (tile base added per tile)
    // and live-plane masks are per-thread constants
    int tc[TL1], tq[TL1], tn2[TL1];
    float2* pk[TL1];
    uint32_t live[TL1];
#pragma unroll
    for (int k = 0; k < TL1; ++k) {
        const int a = tid + k * NT;
        tc[k] = a / (R2 * Q);
        tn2[k] = (a / Q) % R2;
        tq[k] = a % Q;
        pk[k] = X2 + ((int64_t)tc[k] * Kz * plane + (int64_t)tn2[k] * plane + tq[k]);
        uint32_t m = 0;
        for (int n1 = 0; n1 < R1 / 2; ++n1) {
            const int z = R2 * n1 + tn2[k];
            if (z < Kz && __ldg(&planeok[z])) m |= 1u << n1;
        }
        live[k] = m;
    }
    // CTA-uniform fast paths: every kept plane z < Kz = N/2 exists (unpredicated stores) and
    // is non-empty (unpredicated loads)
    const bool full_z = Kz == P::NH;
    bool dense_z = full_z;
    for (int z = 0; z < Kz; ++z) dense_z = dense_z && __ldg(&planeok[z]) != 0;
    // L2 role and its twiddles W_N^{n2 k1}, n2 = 1 .. R2-1
    const bool l2 = tid < NL2;
    const int k1 = tid / Q, q2 = tid % Q;
    float2 w2[R2];
#pragma unroll
    for (int m = 0; m < R2; ++m) w2[m] = l2 ? __ldg(&tw[(m * k1) & (N - 1)]) : zero;
    if constexpr (DM > 0) {
        // the mode-3 factor rows of the octant (kh <= N/2) are the same for every unit: on chip once
        for (int e = tid; e < 7 * NK * DM; e += NT) {
            const int m = e / (NK * DM), rest = e - m * NK * DM, kh = rest / DM, c = rest - kh * DM;
            const int d3 = sv.rk[m][2];
            F3s[e] = c < d3 ? __ldg(&sv.fac[m][2][(int64_t)kh * d3 + c]) : 0.f;
        }
    }
    // tile walk without divisions: unit u = (oy, xt); within a unit the row (ky = oy, then
    // Ny - oy) and, fastest, the RHS r.  base = element offset of (r, c = 0, z = 0, ky, xt * Q)
    const int64_t rstride = (int64_t)5 * Kz * plane;
    auto rows_of = [&](int o) { return (o == 0 || 2 * o == Ny) ? 1 : 2; };
    auto base_of = [&](int o, int x, int rw, int rr) -> int64_t {
        return (int64_t)rr * rstride + (int64_t)(rw == 0 ? o : Ny - o) * Nxs + x * Q;
    };
    const int64_t zstep = (int64_t)R2 * plane;
    float2 nx[TL1][R1 / 2];   // prefetch of the next tile's live inputs
    auto load_tile = [&](int64_t b) {
#pragma unroll
        for (int k = 0; k < TL1; ++k) {
            const float2* src = pk[k] + b;
            if (dense_z) {
#pragma unroll
                for (int n1 = 0; n1 < R1 / 2; ++n1) {
                    nx[k][n1] = *src;
                    src += zstep;
                }
            } else {
#pragma unroll
                for (int n1 = 0; n1 < R1 / 2; ++n1) {
                    nx[k][n1] = ((live[k] >> n1) & 1u) ? *src : zero;
                    src += zstep;
                }
            }
        }
    };
    int u = u0, oy = u0 / tiles_x, xt = u0 - (u0 / tiles_x) * tiles_x, row = 0, r = 0;
    // folded moment-form constants, applied once per unit when KV is built:
    // g K0, gx K1x, g K1y (its ky sign at use), -2g K1z (its kz sign at use), g K2x, g K2y, 4g K2z
    auto kv_scale = [&](int m, int q) -> float {
        const int kx = kxg + xt * Q + q;
        return m == 1 ? (kx <= (Nx >> 1) ? g : -g) : m == 3 ? -2.f * g : m == 6 ? 4.f * g : g;
    };
    int64_t base = 0;
    if (u < u1) {
        base = base_of(oy, xt, 0, 0);
        load_tile(base);
    }
    int cur_oy = -1;
    for (int s = 0; u < u1; ++s) {
        float2* Tb = T + (NBUF == 2 ? (s & 1) * TE : 0);
        const int ky = row == 0 ? oy : Ny - oy;
        if (row == 0 && r == 0) {
            // the unit's raw kernel spectra KV[kh][q][m] (the previous tile's L2 finished at its barrier)
            if constexpr (DM > 0) {
                if (oy != cur_oy) {
                    // G_m = core_m x2 F2_m[oy]   ([c3][c1], once per oy; zero outside the ranks)
                    __syncthreads();   // (first unit: F3s; later: the previous unit's H reads of G)
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
                // H_m[q] = G_m x1 F1_m[ox_q]: one task per (m, q), the factor row in registers
                for (int t = tid; t < 7 * Q; t += NT) {
                    const int m = t / Q, q = t - m * Q;
                    const int d1 = sv.rk[m][0];
                    const int kx = kxg + xt * Q + q;
                    const int ox = kx <= (Nx >> 1) ? kx : Nx - kx;
                    const float* f1 = sv.fac[m][0] + (int64_t)ox * d1;
                    float fr[DM];
#pragma unroll
                    for (int c = 0; c < DM; ++c) fr[c] = c < d1 ? __ldg(&f1[c]) : 0.f;
                    const float* Gm = G + m * DM * DP;
                    float* hq = H + (m * Q + q) * DP;
#pragma unroll 4
                    for (int c3 = 0; c3 < DM; ++c3) {
                        float acc = 0.f;
#pragma unroll
                        for (int c = 0; c < DM; ++c) acc = fmaf(Gm[c3 * DP + c], fr[c], acc);
                        hq[c3] = acc;
                    }
                }
                __syncthreads();
                // KV[kh][q][m] = F3_m[kh] . H_m[q]: a thread keeps its column's H row in registers
                // (q = tid mod Q is fixed, NT is a multiple of Q) and walks kh; F3 rows by 16-byte loads
                static_assert(NT % Q == 0 && DM % 4 == 0, "KV build: fixed column per thread");
                {
                    const int q = tid % Q;
#pragma unroll 1
                    for (int m = 0; m < 7; ++m) {
                        const float* F3m = F3s + m * NK * DM;
                        const float* hq = H + (m * Q + q) * DP;
                        const float sc = kv_scale(m, q);
                        float hr[DM];
#pragma unroll
                        for (int c = 0; c < DM; ++c) hr[c] = hq[c];
                        for (int kh = tid / Q; kh < NK; kh += NT / Q) {
                            const float4* f3 = reinterpret_cast<const float4*>(F3m + kh * DM);
                            float acc = 0.f;
#pragma unroll
                            for (int c4 = 0; c4 < DM / 4; ++c4) {
                                const float4 f = f3[c4];
                                acc = fmaf(f.x, hr[4 * c4], acc);
                                acc = fmaf(f.y, hr[4 * c4 + 1], acc);
                                acc = fmaf(f.z, hr[4 * c4 + 2], acc);
                                acc = fmaf(f.w, hr[4 * c4 + 3], acc);
                            }
                            KV[(kh * Q + q) * KVS + m] = sc * acc;
                        }
                    }
                }
            } else {
                const int64_t pl = (int64_t)sv.hx * sv.hy * sv.hz;
                for (int t = tid; t < 7 * NK * Q; t += NT) {
                    const int q = t % Q, rest = t / Q;
                    const int kh = rest % NK, m = rest / NK;
                    const int kx = kxg + xt * Q + q;
                    const int ox = kx <= (Nx >> 1) ? kx : Nx - kx;
                    KV[(kh * Q + q) * KVS + m] =
                        kv_scale(m, q) * __ldg(&sv.spec[m * pl + ((int64_t)kh * sv.hy + oy) * sv.hx + ox]);
                }
            }
            // published to L2 by the barrier after L1
        }
        // next tile of this CTA
        int un = u, oyn = oy, xtn = xt, rown = row, rn = r + 1;
        if (rn == nrhs) {
            rn = 0;
            if (++rown == rows_of(oy)) {
                rown = 0;
                ++un;
                if (++xtn == tiles_x) {
                    xtn = 0;
                    ++oyn;
                }
            }
        }
        const int64_t basen = base_of(oyn, xtn, rown, rn);
        // L1 forward
#pragma unroll
        for (int k = 0; k < TL1; ++k) {
            float2 v[R1];
#pragma unroll
            for (int n1 = 0; n1 < R1; ++n1) v[n1] = n1 < R1 / 2 ? nx[k][n1] : zero;
            reg_fft<R1, -1, true>(v);
            float2* t1 = Tb + (tc[k] * R2 + tn2[k]) * TB + tq[k];
#pragma unroll
            for (int kk = 0; kk < R1; ++kk) t1[kk * Q] = v[kk];
        }
        // the next tile's inputs: in flight during L2 and the inverse L1 of this tile
        if (un < u1) load_tile(basen);
        __syncthreads();
        // L2: twiddle, R2-point FFT, MAC, inverse, twiddle
        if (l2) {
            const uint32_t sy = ky <= (Ny >> 1) ? 0u : 0x80000000u;   // K1y is odd in ky
            float2 uu[5][R2];
#pragma unroll
            for (int c = 0; c < 5; ++c) {
#pragma unroll
                for (int m = 0; m < R2; ++m) {
                    const float2 x = Tb[(c * R2 + m) * TB + k1 * Q + q2];
                    uu[c][m] = m ? cmul(x, w2[m]) : x;
                }
                reg_fft<R2, -1>(uu[c]);
            }
#pragma unroll
            for (int k2 = 0; k2 < R2; ++k2) {
                const int kz = k1 + R1 * k2;
                const int kh = kz <= (N >> 1) ? kz : N - kz;
                const uint32_t s3 = kz <= (N >> 1) ? 0u : 0x80000000u;   // K1z is odd in kz
                const float4 ka = *reinterpret_cast<const float4*>(KV + (kh * Q + q2) * KVS);
                const float4 kb = *reinterpret_cast<const float4*>(KV + (kh * Q + q2) * KVS + 4);
                // the constants were folded into KV; only the two odd-axis signs are applied here
                const float f0 = ka.x, f1 = ka.y, f2 = __uint_as_float(__float_as_uint(ka.z) ^ sy);
                const float f3 = __uint_as_float(__float_as_uint(ka.w) ^ s3);
                const float f4 = kb.x, f5 = kb.y, f6 = kb.z;
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
                    Tb[(c * R2 + m) * TB + k1 * Q + q2] = m ? cmul(uu[c][m], wc) : uu[c][m];
                }
            }
        }
        __syncthreads();
        // L1 inverse: z = n2 + R2 n1, kept z < Kz, straight to HBM
#pragma unroll
        for (int k = 0; k < TL1; ++k) {
            float2 v[R1];
            const float2* t1 = Tb + (tc[k] * R2 + tn2[k]) * TB + tq[k];
#pragma unroll
            for (int kk = 0; kk < R1; ++kk) v[kk] = t1[kk * Q];
            reg_fft<R1, +1>(v);
            float2* dst = pk[k] + base;
            if (full_z) {
#pragma unroll
                for (int n1 = 0; n1 < R1 / 2; ++n1) {
                    *dst = v[n1];
                    dst += zstep;
                }
            } else {
#pragma unroll
                for (int n1 = 0; n1 < R1 / 2; ++n1) {
                    if (R2 * n1 + tn2[k] < Kz) *dst = v[n1];
                    dst += zstep;
                }
            }
        }
        u = un;
        oy = oyn;
        xt = xtn;
        row = rown;
        r = rn;
        base = basen;
        // no barrier here even with one T buffer: the next tile's forward L1 writes, task by task,
        // exactly the T pencils (c, n2, q) this thread has just read in the inverse L1
    }
}

}  // namespace svh
