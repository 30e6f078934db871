// Fused-exchange variant of the slab-decomposed matvec (SURVEY 8(e)(2) "then a fused variant";
// the operator is Eq. 9).  Instead of packing the x-transformed current into a local
// send buffer and handing it to an all-to-all, the pack kernel stores each destination's chunk
// straight into that peer's receive buffer through NVLink peer memory (CUDA IPC mappings), then
// every rank signals its peers and waits for theirs with stream memory operations:
//   signal: cuStreamWriteValue32(peer_flags[p] + slot P + rank, epoch)   (preceded by a full
//           memory barrier, so the peer sees the chunk before the flag)
//   wait:   cuStreamWaitValue32(own_flags + slot P + s, epoch, GEQ) for every s
// The wait blocks the STREAM, not an SM: no kernel spins on a flag, so ranks that share a GPU
// (the tests) or are scheduled in any order cannot deadlock.  The local send write, its
// re-read by the collective and the collective's launch disappear from the product.
//
// Buffers (caller-owned, from svh_ipc_alloc; peers open them with svh_ipc_open):
//   recv1, recv2 : [s][nrhs][5][Kz][Kyl][Nxl] complex64 per rank (chunk s written by rank s);
//                  recv1 takes the forward exchange, recv2 the middle one, so an exchange never
//                  overwrites a buffer its owner may still be reading
//   flags        : uint32 [2][P] per rank (slot 0 = forward, 1 = middle), zero-initialised;
//                  epochs increase by one per product
#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>

#include <cuda.h>
#include <cuda_runtime.h>

#include "internal.h"

namespace svh {
namespace {

constexpr int kMaxPeers = 8;
struct PeerPtrs {
    float2* p[kMaxPeers];
};

// element (p, b, y, k) of the exchange <-> X1 element b*SB + y*SY + p*SP + k; stored at
// dst.p[p] + rank * chunk + (b * Kyl + y) * Nxl + k (the chunk this rank owns in p's buffer)
__global__ void k_slab_push(PeerPtrs dst, const float2* __restrict__ X1, int P, int rank, int64_t Bt, int Kyl, int Nxl,
                            int64_t SB, int64_t SY, int64_t SP) {
    const int64_t per = Bt * Kyl * Nxl;   // one chunk
    const int64_t total = (int64_t)P * per;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(i % Nxl);
        int64_t r = i / Nxl;
        const int y = (int)(r % Kyl);
        r /= Kyl;
        const int64_t b = r % Bt;
        const int p = (int)(r / Bt);
        const float2 v = X1[b * SB + (int64_t)y * SY + (int64_t)p * SP + k];
        dst.p[p][(int64_t)rank * per + i - (int64_t)p * per] = v;
    }
}

using WriteFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using WaitFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

template <typename F>
F driver_fn(const char* name) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return reinterpret_cast<F>(p);
}

void exchange(svh_handle* h, int rank, int P, const PeerPtrs& dst, uint32_t* const* peer_flags, uint32_t* own_flags,
              int slot, uint32_t epoch, int64_t Bt, int Kyl, int Nxl, int64_t SB, int64_t SY, int64_t SP,
              cudaStream_t s) {
    static WriteFn wr = nullptr;
    static WaitFn wt = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        wr = driver_fn<WriteFn>("cuStreamWriteValue32");
        wt = driver_fn<WaitFn>("cuStreamWaitValue32");
    });
    SVH_CHECK(wr && wt, SVH_ECUDA, "stream memory operations (cuStreamWrite/WaitValue32) unavailable");
    const int64_t total = (int64_t)P * Bt * Kyl * Nxl;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, (int64_t)nsm * 8));
    SVH_LAUNCH(k_slab_push, grid, 256, 0, s, dst, h->X1, P, rank, Bt, Kyl, Nxl, SB, SY, SP);
    for (int p = 0; p < P; ++p) {
        const CUresult r = wr((CUstream)s, (CUdeviceptr)(peer_flags[p] + slot * P + rank), epoch, 0);
        SVH_CHECK(r == CUDA_SUCCESS, SVH_ECUDA, "cuStreamWriteValue32 failed: " + std::to_string((int)r));
    }
    for (int q = 0; q < P; ++q) {
        const CUresult r = wt((CUstream)s, (CUdeviceptr)(own_flags + slot * P + q), epoch, CU_STREAM_WAIT_VALUE_GEQ);
        SVH_CHECK(r == CUDA_SUCCESS, SVH_ECUDA, "cuStreamWaitValue32 failed: " + std::to_string((int)r));
    }
}

PeerPtrs peers(void* const* bufs, int P) {
    PeerPtrs d{};
    for (int p = 0; p < P; ++p) {
        SVH_CHECK(bufs[p] != nullptr, SVH_EINVAL, "null peer buffer");
        d.p[p] = static_cast<float2*>(bufs[p]);
    }
    return d;
}

}  // namespace

void slab_forward_p2p(svh_handle* h, int rank, int P, const float2* I, void* const* recv1_peers,
                      uint32_t* const* flag_peers, uint32_t epoch, int nrhs, cudaStream_t s) {
    SVH_CHECK(P >= 1 && P <= kMaxPeers, SVH_EINVAL, "P2P slab exchange: 1 <= P <= 8");
    slab_forward_compute(h, rank, P, I, nrhs, s);
    const int Kyl = h->ky / P, Nxl = h->nx / P;
    const int64_t Bt = 5LL * nrhs * h->kz;
    exchange(h, rank, P, peers(recv1_peers, P), flag_peers, flag_peers[rank], 0, epoch, Bt, Kyl, Nxl,
             (int64_t)Kyl * h->nx, h->nx, Nxl, s);
}

void slab_middle_p2p(svh_handle* h, int rank, int P, const float2* recv1, void* const* recv2_peers,
                     uint32_t* const* flag_peers, uint32_t epoch, int nrhs, cudaStream_t s) {
    SVH_CHECK(P >= 1 && P <= kMaxPeers, SVH_EINVAL, "P2P slab exchange: 1 <= P <= 8");
    slab_middle_compute(h, rank, P, recv1, nrhs, s);
    const int Kyl = h->ky / P, Nxl = h->nx / P;
    const int64_t Bt = 5LL * nrhs * h->kz;
    exchange(h, rank, P, peers(recv2_peers, P), flag_peers, flag_peers[rank], 1, epoch, Bt, Kyl, Nxl,
             (int64_t)h->ky * Nxl, Nxl, (int64_t)Kyl * Nxl, s);
}

}  // namespace svh

using namespace svh;
extern "C" {

int svh_ipc_alloc(size_t bytes, void** dptr, void* handle) {
    try {
        SVH_CHECK(dptr && handle && bytes > 0, SVH_EINVAL, "bad ipc alloc args");
        *dptr = nullptr;
        if (cudaMalloc(dptr, bytes) != cudaSuccess) {
            cudaGetLastError();
            throw Error{SVH_ENOMEM, "ipc buffer allocation failed"};
        }
        SVH_CUDA(cudaMemset(*dptr, 0, bytes));
        cudaIpcMemHandle_t hd;
        SVH_CUDA(cudaIpcGetMemHandle(&hd, *dptr));
        static_assert(sizeof(hd) == 64, "cudaIpcMemHandle_t is 64 bytes");
        std::memcpy(handle, &hd, sizeof(hd));
        return SVH_OK;
    }
    SVH_C_ABI_CATCH
}

int svh_ipc_free(void* dptr) {
    try {
        SVH_CUDA(cudaFree(dptr));
        return SVH_OK;
    }
    SVH_C_ABI_CATCH
}

int svh_ipc_open(const void* handle, void** dptr) {
    try {
        SVH_CHECK(handle && dptr, SVH_EINVAL, "bad ipc open args");
        cudaIpcMemHandle_t hd;
        std::memcpy(&hd, handle, sizeof(hd));
        SVH_CUDA(cudaIpcOpenMemHandle(dptr, hd, cudaIpcMemLazyEnablePeerAccess));
        return SVH_OK;
    }
    SVH_C_ABI_CATCH
}

int svh_ipc_close(void* dptr) {
    try {
        SVH_CUDA(cudaIpcCloseMemHandle(dptr));
        return SVH_OK;
    }
    SVH_C_ABI_CATCH
}

int svh_slab_forward_p2p(svh_handle* h, int32_t rank, int32_t P, const void* I_slab, void* const* recv1_peers,
                         uint32_t* const* flag_peers, uint32_t epoch, int32_t nrhs, svh_stream stream) {
    try {
        SVH_CHECK(h && I_slab && recv1_peers && flag_peers && nrhs >= 1 && epoch > 0, SVH_EINVAL, "bad p2p slab args");
        SVH_CUDA(cudaSetDevice(h->device));
        slab_forward_p2p(h, rank, P, (const float2*)I_slab, recv1_peers, flag_peers, epoch, nrhs, (cudaStream_t)stream);
        return SVH_OK;
    }
    SVH_C_ABI_CATCH
}

int svh_slab_middle_p2p(svh_handle* h, int32_t rank, int32_t P, const void* recv1, void* const* recv2_peers,
                        uint32_t* const* flag_peers, uint32_t epoch, int32_t nrhs, svh_stream stream) {
    try {
        SVH_CHECK(h && recv1 && recv2_peers && flag_peers && nrhs >= 1 && epoch > 0, SVH_EINVAL, "bad p2p slab args");
        SVH_CUDA(cudaSetDevice(h->device));
        slab_middle_p2p(h, rank, P, (const float2*)recv1, recv2_peers, flag_peers, epoch, nrhs, (cudaStream_t)stream);
        return SVH_OK;
    }
    SVH_C_ABI_CATCH
}

}  // extern "C"
