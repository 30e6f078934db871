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

__host__ __device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__host__ __device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__host__ __device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__host__ __device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
// multiply by i*s (s real)
__host__ __device__ __forceinline__ float2 cmul_i(float2 a, float s) { return make_float2(-a.y * s, a.x * s); }

inline int ilog2(int64_t n) {
    int l = 0;
    while ((int64_t(1) << l) < n) ++l;
    return l;
}

}  // namespace svh
