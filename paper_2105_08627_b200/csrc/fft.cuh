// Radix-2^k FFT building blocks for the matvec passes (Eq. 9 FFT/IFFT).
//
// * reg_fft<L, DIR>: length-L (L <= 64, power of two) FFT of a register array,
//   fully unrolled; twiddles are compile-time constants (twiddle64.h).
// * smem_fft<N, DIR>: length-N (N <= 4096) FFT of Q pencils held in shared
//   memory at S[j * PP + q] (element j of pencil q).  Two-level Cooley-Tukey
//   N = R1 * R2: phase 1 = R2*Q tasks each doing an R1-point register FFT and
//   the W_N^{n2 k1} twiddle, transposed through shared memory; phase 2 =
//   R1*Q tasks each doing an R2-point register FFT.  Requires
//   blockDim.x >= max(R1, R2) * Q.  Output is in natural order.
// DIR = -1: forward exp(-2 pi i jk/N); DIR = +1: inverse (unscaled).
#pragma once
#include "common.cuh"
#include "twiddle64.h"

#include <utility>

namespace svh {

__host__ __device__ constexpr int brev_c(int i, int L) {
    int r = 0;
    for (int b = 1; b < L; b <<= 1) {
        r = (r << 1) | (i & 1);
        i >>= 1;
    }
    return r;
}

// compile-time loop: f(std::integral_constant<int, i>) for i < N (keeps register
// arrays in registers: every index below is a constant expression)
template <typename F, int... Is>
__device__ __forceinline__ void static_for_impl(F&& f, std::integer_sequence<int, Is...>) {
    (f(std::integral_constant<int, Is>{}), ...);
}
template <int N, typename F>
__device__ __forceinline__ void static_for(F&& f) {
    static_for_impl(f, std::make_integer_sequence<int, N>{});
}

__host__ __device__ constexpr int ilog2_c(int n) { return n <= 1 ? 0 : 1 + ilog2_c(n >> 1); }

// HALF_IN: inputs L/2..L-1 are known zero (the zero-padded half of a circulant
// embedding).  After the bit reversal they sit at the odd positions, so the
// first radix-2 stage reduces to copies (x + 0 is not folded by the compiler under
// IEEE semantics, so the pruning is explicit).
template <int L, int DIR, bool HALF_IN = false>
__device__ __forceinline__ void reg_fft(float2 (&v)[L]) {
    if constexpr (L > 1) {
        static_for<L>([&](auto I) {
            constexpr int i = decltype(I)::value;
            constexpr int j = brev_c(i, L);
            if constexpr (j > i) {
                const float2 t = v[i];
                v[i] = v[j];
                v[j] = t;
            }
        });
        static_for<ilog2_c(L)>([&](auto S) {
            constexpr int len = 2 << decltype(S)::value;
            constexpr int half = len >> 1;
            static_for<L / len>([&](auto B) {
                constexpr int i = decltype(B)::value * len;
                static_for<half>([&](auto Kc) {
                    constexpr int k = decltype(Kc)::value;
                    const float2 a = v[i + k];
                    const float2 b = v[i + k + half];
                    if constexpr (HALF_IN && len == 2) {
                        v[i + k + half] = a;
                        return;
                    }
                    float2 t;
                    if constexpr (k == 0) {
                        t = b;
                    } else if constexpr (4 * k == len) {
                        // w = exp(DIR * i pi/2) = DIR * i
                        t = DIR < 0 ? make_float2(b.y, -b.x) : make_float2(-b.y, b.x);
                    } else {
                        constexpr float wr = (float)kTwCos64[k * (64 / len)];
                        constexpr float wi = (float)(DIR * kTwSin64[k * (64 / len)]);
                        t = cmul(b, make_float2(wr, wi));
                    }
                    v[i + k] = cadd(a, t);
                    v[i + k + half] = csub(a, t);
                });
            });
        });
    }
}

__host__ __device__ constexpr int fft_r1(int N) {
    if (N <= 64) return N;
    int l = 0;
    while ((1 << l) < N) ++l;
    return 1 << ((l + 1) / 2);
}
__host__ __device__ constexpr int fft_r2(int N) { return N / fft_r1(N); }
// threads needed per pencil by smem_fft (1 when the whole FFT fits one thread)
__host__ __device__ constexpr int fft_threads_per_pencil(int N) {
    return fft_r2(N) == 1 ? 1 : (fft_r1(N) > fft_r2(N) ? fft_r1(N) : fft_r2(N));
}
// max CTA size a pass kernel is compiled for (64-point register FFTs need > 128 regs)
__host__ __device__ constexpr int fft_max_threads(int N) { return fft_r1(N) >= 64 ? 256 : 512; }

// twN[j] = exp(-2 pi i j / N) (fp64-accurate table, rounded to fp32), j < N.
template <int N, int DIR>
__device__ __forceinline__ void smem_fft(float2* S, int PP, int Q, const float2* __restrict__ twN) {
    constexpr int R1 = fft_r1(N);
    constexpr int R2 = fft_r2(N);
    const int tid = threadIdx.x;
    if constexpr (N == 1) {
        return;
    } else if constexpr (R2 == 1) {
        // whole transform in registers: one task per pencil
        if (tid < Q) {
            float2 v[R1];
#pragma unroll
            for (int n = 0; n < R1; ++n) v[n] = S[n * PP + tid];
            reg_fft<R1, DIR>(v);
#pragma unroll
            for (int k = 0; k < R1; ++k) S[k * PP + tid] = v[k];
        }
        __syncthreads();
    } else {
        {
            const bool active = tid < R2 * Q;
            const int n2 = tid / Q, q = tid - (tid / Q) * Q;
            float2 v[R1];
            if (active) {
#pragma unroll
                for (int n1 = 0; n1 < R1; ++n1) v[n1] = S[(R2 * n1 + n2) * PP + q];
                reg_fft<R1, DIR>(v);
#pragma unroll
                for (int k1 = 1; k1 < R1; ++k1) {
                    float2 w = __ldg(&twN[n2 * k1]);
                    if (DIR > 0) w.y = -w.y;
                    v[k1] = cmul(v[k1], w);
                }
            }
            __syncthreads();
            if (active) {
#pragma unroll
                for (int k1 = 0; k1 < R1; ++k1) S[(n2 * R1 + k1) * PP + q] = v[k1];
            }
        }
        __syncthreads();
        {
            const bool active = tid < R1 * Q;
            const int k1 = tid / Q, q = tid - (tid / Q) * Q;
            float2 u[R2];
            if (active) {
#pragma unroll
                for (int n2 = 0; n2 < R2; ++n2) u[n2] = S[(n2 * R1 + k1) * PP + q];
                reg_fft<R2, DIR>(u);
            }
            __syncthreads();
            if (active) {
#pragma unroll
                for (int k2 = 0; k2 < R2; ++k2) S[(k1 + R1 * k2) * PP + q] = u[k2];
            }
        }
        __syncthreads();
    }
}

}  // namespace svh
