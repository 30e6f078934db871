// Shared helpers of libsvh (CUDA side): error handling, complex arithmetic,
// launch accounting.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>

#include "svh.h"

namespace svh {

void set_error(const std::string& msg);
int64_t& launch_counter();

struct Error {
    int code;
    std::string msg;
};

#define SVH_CUDA(call)                                                                       \
    do {                                                                                     \
        cudaError_t e__ = (call);                                                            \
        if (e__ != cudaSuccess) {                                                            \
            throw ::svh::Error{SVH_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e__) \
                                              + " (" + __FILE__ + ":" + std::to_string(__LINE__) + ")"}; \
        }                                                                                    \
    } while (0)

#define SVH_CHECK(cond, code, msg)                \
    do {                                          \
        if (!(cond)) throw ::svh::Error{code, msg}; \
    } while (0)

// every kernel launch in the library goes through this macro (launch accounting
// for bench.py's gpu_launches and for the smoke test)
#define SVH_LAUNCH(kernel, grid, block, smem, stream, ...)                     \
    do {                                                                       \
        kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);            \
        ++::svh::launch_counter();                                             \
        cudaError_t e__ = cudaGetLastError();                                  \
        if (e__ != cudaSuccess)                                                \
            throw ::svh::Error{SVH_ECUDA, std::string("launch ") + #kernel + ": " + \
                                              cudaGetErrorString(e__)};        \
    } while (0)

// Complex arithmetic on float2.  On sm_100a the paired-FP32 instructions
// (FADD2 / FMUL2 / FFMA2, CUDA 12.9 __fadd2_rn etc.) do the real and imaginary
// halves in one instruction; a complex multiply is FMUL2 + FFMA2 with scalar
// broadcast operands.  Measured slower on B200 for these passes (fewer issue
// slots but extra operand moves), so it is opt-in: -DSVH_USE_F32X2.
#if defined(SVH_USE_F32X2) && defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 1000
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return __ffma2_rn(make_float2(a.x, a.x), b, __fmul2_rn(make_float2(a.y, a.y), make_float2(-b.y, b.x)));
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return __fmul2_rn(a, make_float2(s, s)); }
// a * (i s), s real
__device__ __forceinline__ float2 cmul_i(float2 a, float s) {
    return __fmul2_rn(make_float2(a.y, a.x), make_float2(-s, s));
}
// a + b * s (s real)
__device__ __forceinline__ float2 cfma_s(float2 b, float s, float2 a) { return __ffma2_rn(b, make_float2(s, s), a); }
#else
__host__ __device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__host__ __device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__host__ __device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__host__ __device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
__host__ __device__ __forceinline__ float2 cmul_i(float2 a, float s) { return make_float2(-a.y * s, a.x * s); }
__host__ __device__ __forceinline__ float2 cfma_s(float2 b, float s, float2 a) {
    return make_float2(a.x + b.x * s, a.y + b.y * s);
}
#endif

inline int ilog2(int64_t n) {
    int l = 0;
    while ((int64_t(1) << l) < n) ++l;
    return l;
}

}  // namespace svh
