// Shared helpers of libsvh (CUDA side): error handling, complex arithmetic,
// launch accounting.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <exception>
#include <new>
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

// catch clauses of every extern "C" entry point: no C++ exception crosses the C-ABI
#define SVH_C_ABI_CATCH                                                                   \
    catch (const ::svh::Error& e) {                                                       \
        ::svh::set_error(e.msg);                                                          \
        return e.code;                                                                    \
    }                                                                                     \
    catch (const std::bad_alloc&) {                                                       \
        ::svh::set_error("host allocation failed");                                       \
        return SVH_ENOMEM;                                                                \
    }                                                                                     \
    catch (const std::exception& e) {                                                     \
        ::svh::set_error(e.what());                                                       \
        return SVH_EINVAL;                                                                \
    }

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

// Complex arithmetic on float2 (re, im).  In device code for sm_100a every helper is
// one or two paired-FP32 instructions (FADD2 / FMUL2 / FFMA2 act on both halves of a
// 64-bit register pair): the swap (a.y, a.x) and scalar broadcasts fold into operand
// modifiers (.LO_HI, .F32), so a complex multiply is FMUL2 + FFMA2 and a butterfly
// add/sub one FADD2 each -- about 0.55x the FP instructions of the scalar form on the
// FFT-bound passes (cuobjdump-checked).  -DSVH_SCALAR_COMPLEX
// restores the scalar forms.
#if !defined(SVH_SCALAR_COMPLEX) && defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 1000
#define SVH_F32X2 1
#endif
__host__ __device__ __forceinline__ float2 cswap(float2 a) { return make_float2(a.y, a.x); }
__host__ __device__ __forceinline__ float2 cadd(float2 a, float2 b) {
#ifdef SVH_F32X2
    return __fadd2_rn(a, b);
#else
    return make_float2(a.x + b.x, a.y + b.y);
#endif
}
__host__ __device__ __forceinline__ float2 csub(float2 a, float2 b) {
#ifdef SVH_F32X2
    return __fadd2_rn(a, make_float2(-b.x, -b.y));
#else
    return make_float2(a.x - b.x, a.y - b.y);
#endif
}
__host__ __device__ __forceinline__ float2 cmul(float2 a, float2 b) {
#ifdef SVH_F32X2
    // (a.x b.x - a.y b.y, a.y b.x + a.x b.y) = a*(b.x, b.x) + swap(a)*(-b.y, b.y)
    return __ffma2_rn(cswap(a), make_float2(-b.y, b.y), __fmul2_rn(a, make_float2(b.x, b.x)));
#else
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
#endif
}
__host__ __device__ __forceinline__ float2 cscale(float2 a, float s) {
#ifdef SVH_F32X2
    return __fmul2_rn(a, make_float2(s, s));
#else
    return make_float2(a.x * s, a.y * s);
#endif
}
// a * (i s), s real
__host__ __device__ __forceinline__ float2 cmul_i(float2 a, float s) {
#ifdef SVH_F32X2
    return __fmul2_rn(cswap(a), make_float2(-s, s));
#else
    return make_float2(-a.y * s, a.x * s);
#endif
}
// a + b * s (s real)
__host__ __device__ __forceinline__ float2 cfma_s(float2 b, float s, float2 a) {
#ifdef SVH_F32X2
    return __ffma2_rn(b, make_float2(s, s), a);
#else
    return make_float2(a.x + b.x * s, a.y + b.y * s);
#endif
}

inline int ilog2(int64_t n) {
    int l = 0;
    while ((int64_t(1) << l) < n) ++l;
    return l;
}

}  // namespace svh
