// Strided passes B (forward y-FFT, zero-padded) and D (inverse y-FFT, cropped) of the matvec
// (Eq. 9) for Ny = 1024 / 2048: the Stockham radix-16 FFT of rowfft.cuh applied to Q
// pencils at once.
//
// Tile = Q consecutive kx of one non-empty plane p = rc Kz + z.  Its input rows (B: the Ky rows
// of X1, D: the Ny rows of X2) stream HBM -> shared memory by TMA (cp.async.bulk.tensor, box
// Q x 256 rows) into an S-deep mbarrier ring, so the next tiles' loads are in flight while this
// one is transformed; stage 0 reads the dense staged tile, stages 1-2 run in place on one padded
// work buffer W (element (i, q) at rpad(i) Q + q: conflict-free for every stage), and the last
// stage stores to HBM (B: all Ny rows of X2, staged in shared memory and written by TMA stores;
// D: straight from registers, the rows y < Ky that hold a voxel, the only ones pass E reads).  B zeroes the staged rows that hold no voxel (pass A never
// wrote them) and the rows Ky <= y < Ny/2 (outside the box: TMA zero fill).
#pragma once
#include "rowfft.cuh"
#include "tma.cuh"

namespace svh {

template <int N, int Q, int DIR>
struct YPlan {
    static_assert(N == 1024 || N == 2048, "y plan: N = 1024 or 2048");
    static constexpr int T = N / 16;              // threads per pencil
    static constexpr int NT = T * Q;
    static constexpr int RL = N / 256;            // last-stage radix (stages 16 x 16 x RL)
    static constexpr int PADN = N + N / 16;
    static constexpr int SR = DIR < 0 ? N / 2 : N;   // staged rows
    static constexpr int BOX = 256;
    static constexpr int S = 2;                   // ring depth
    static constexpr size_t stage_b = (size_t)SR * Q * sizeof(float2);
    static constexpr size_t W_b = (size_t)PADN * Q * sizeof(float2);
    static constexpr int MW = (N / 2 + 31) / 32;  // row-mask words of a plane (y < N/2)
    // forward: the output tile (Ny rows x Q, dense) is staged for TMA stores
    static constexpr size_t O_b = DIR < 0 ? (size_t)N * Q * sizeof(float2) : 0;
    static constexpr size_t smem = S * stage_b + W_b + O_b + (size_t)S * MW * 4 + S * 8 + 64;
};

template <int N, int Q, int DIR>
__global__ void __launch_bounds__(YPlan<N, Q, DIR>::NT, 1)
    k_ypass(float2* __restrict__ out, const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout,
            const float2* __restrict__ tw,
            int Nx, int Kz, int Lin, int Lout, int ntiles, int tiles_x, const int32_t* __restrict__ planes, int nzp,
            const uint32_t* __restrict__ rowmask, int rowMW) {
    using P = YPlan<N, Q, DIR>;
    constexpr int T = P::T, NT = P::NT, RL = P::RL, SR = P::SR, BOX = P::BOX, S = P::S, MW = P::MW;
    extern __shared__ __align__(128) unsigned char smraw[];
    float2* stage = reinterpret_cast<float2*>(smraw);
    float2* W = reinterpret_cast<float2*>(smraw + S * P::stage_b);
    float2* O = reinterpret_cast<float2*>(smraw + S * P::stage_b + P::W_b);
    uint32_t* M = reinterpret_cast<uint32_t*>(smraw + S * P::stage_b + P::W_b + P::O_b);
    uint64_t* bar =
        reinterpret_cast<uint64_t*>(smraw + ((S * P::stage_b + P::W_b + P::O_b + S * MW * 4 + 7) / 8) * 8);
    const int tid = threadIdx.x;
    const int j = tid / Q, q = tid % Q;
    const float2 zero = make_float2(0.f, 0.f);
    if (tid == 0) {
        for (int st = 0; st < S; ++st) mbar_init(&bar[st], 1);
        mbar_fence_init();
    }
    __syncthreads();
    auto decode = [&](int t, int& z, int& p, int& x0) {
        const int xt = t % tiles_x, pr = t / tiles_x;
        const int rc = pr / nzp;
        z = __ldg(&planes[pr - rc * nzp]);
        p = rc * Kz + z;
        x0 = xt * Q;
    };
    // thread 0: TMA of tile t into slot st (+ the plane's row-mask words)
    auto issue = [&](int t, int st) {
        if (t >= ntiles) return;
        int z, p, x0;
        decode(t, z, p, x0);
        mbar_arrive_expect_tx(&bar[st], (uint32_t)P::stage_b);
#pragma unroll
        for (int b = 0; b < SR / BOX; ++b) tma_load_3d(stage + st * SR * Q + b * BOX * Q, &tin, x0, b * BOX, p, &bar[st]);
    };
    auto load_mask = [&](int t, int st) {
        if (t >= ntiles) return;
        int z, p, x0;
        decode(t, z, p, x0);
        for (int w = tid; w < MW; w += NT) M[st * MW + w] = w < rowMW ? __ldg(&rowmask[(int64_t)z * rowMW + w]) : 0u;
    };
    // stage-1 twiddles W_256^{k r}, k = j mod 16 (per-thread constants)
    float2 w1[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) w1[r] = tw_at<DIR>(tw, ((j & 15) * r * (N / 256)) & (N - 1));
    int t = blockIdx.x;
    if (tid == 0)
        for (int st = 0; st < S; ++st) issue(t + st * (int)gridDim.x, st);
    for (int st = 0; st < S; ++st) load_mask(t + st * (int)gridDim.x, st);
    for (int i = 0; t < ntiles; ++i, t += gridDim.x) {
        const int st = i % S;
        int z, p, x0;
        decode(t, z, p, x0);
        mbar_wait(&bar[st], (uint32_t)((i / S) & 1));
        __syncthreads();   // the previous tile's stage-2 reads of W are done; M[st] visible
        const float2* src = stage + st * SR * Q;
        const uint32_t* Ms = M + st * MW;
        // stage 0: radix 16, Ns = 1; rows n = j + r N/16
        {
            float2 v[16];
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                const int n = j + r * (N / 16);
                if (DIR < 0) {
                    const bool live = r < 8 && n < Lin && ((Ms[n >> 5] >> (n & 31)) & 1u);
                    v[r] = live ? src[n * Q + q] : zero;
                } else {
                    v[r] = src[n * Q + q];
                }
            }
            reg_fft<16, DIR, (DIR < 0)>(v);
#pragma unroll
            for (int r = 0; r < 16; ++r) W[rpad(j * 16 + r) * Q + q] = v[r];
        }
        uint32_t keep = 0;   // inverse: which of this thread's output rows hold a voxel
        if (DIR > 0) {
#pragma unroll
            for (int i2 = 0; i2 < 16 / RL; ++i2)
#pragma unroll
                for (int r = 0; r < RL / 2; ++r) {
                    const int n = j + i2 * T + r * (N / RL);
                    if (n < Lout && ((Ms[n >> 5] >> (n & 31)) & 1u)) keep |= 1u << (i2 * RL + r);
                }
        }
        __syncthreads();   // the staged tile is consumed: refill its slot
        if (tid == 0) issue(t + S * (int)gridDim.x, st);
        load_mask(t + S * (int)gridDim.x, st);
        // stage 1: radix 16, Ns = 16, in place
        {
            float2 v[16];
#pragma unroll
            for (int r = 0; r < 16; ++r) v[r] = W[rpad(j + r * (N / 16)) * Q + q];
            __syncthreads();
            stage_twiddle<16, DIR>(v, w1);
            reg_fft<16, DIR>(v);
            const int base = (j >> 4) * 256 + (j & 15);
#pragma unroll
            for (int r = 0; r < 16; ++r) W[rpad(base + r * 16) * Q + q] = v[r];
        }
        // forward: the previous tile's TMA stores must have read O before stage 2 rewrites it --
        // waited for only here, so stages 0-1 of this tile overlap the drain of those stores
        if (DIR < 0 && tid == 0) tma_store_wait_read0();
        __syncthreads();
        // stage 2 (last): radix RL, Ns = 256, tasks tt = j + i2 T; outputs tt + r N/RL
        float2* dst = out + (int64_t)p * Lout * Nx + x0 + q;
#pragma unroll
        for (int i2 = 0; i2 < 16 / RL; ++i2) {
            const int tt = j + i2 * T;
            float2 v[RL];
#pragma unroll
            for (int r = 0; r < RL; ++r) v[r] = W[rpad(tt + r * (N / RL)) * Q + q];
#pragma unroll
            for (int r = 1; r < RL; ++r) v[r] = cmul(v[r], tw_at<DIR>(tw, (tt * r) & (N - 1)));
            reg_fft<RL, DIR>(v);
#pragma unroll
            for (int r = 0; r < RL; ++r) {
                const int n = tt + r * (N / RL);
                if (DIR < 0)
                    O[n * Q + q] = v[r];
                else if (r < RL / 2 && ((keep >> (i2 * RL + r)) & 1u))
                    dst[(int64_t)n * Nx] = v[r];
            }
        }
        if (DIR < 0) {   // the whole output tile leaves by TMA stores (Ny / 256 boxes)
            fence_proxy_async_smem();
            __syncthreads();
            if (tid == 0) {
#pragma unroll
                for (int b = 0; b < N / BOX; ++b) tma_store_3d(&tout, x0, b * BOX, p, O + b * BOX * Q);
                tma_store_commit();
            }
        }
    }
    if (DIR < 0 && tid == 0) tma_store_wait0();
}

}  // namespace svh
