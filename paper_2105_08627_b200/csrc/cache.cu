// Algorithm 2 (Sec. II.B.1): install-time cache of Tucker-compressed Toeplitz
// tensors, and the setup path that restores the kernels of a grid from it instead of
// evaluating the 6-D interaction integrals (Table II).
//
// Build (once): the 7 unit-voxel kernels (Sec. 3 of DESIGN.md) on a large offset domain
// Nmax_x x Nmax_y x Nmax_z are Tucker-compressed by Algorithm 1 (the same weighted HOSVD
// as the Tucker matvec mode, tucker.cu) and written to disk.  Setup (every run): for a grid
// K_x x K_y x K_z <= Nmax the Toeplitz tensor of the grid is the leading K_x x K_y x K_z
// block, i.e. core x_i U_i[:K_i] (factor rows trimmed, "resizing"), un-weighted; the
// Delta-x^5 scaling of Alg. 2 line 6 is the j*omega*mu0*dx prefactor applied at matvec time
// (App. B, reading G1), so the cached kernels are dx-independent.
//
// File "SVXT" v2 (little endian; the layout of SPEC S:236): header = char magic[4] "SVXT",
// u32 version, f64 tol, u64 nmax[3], u32 block count (7); per block (kernel q = 0..6, in the
// order K0, K1x, K1y, K1z, K2x, K2y, K2z): char tag[2] ("00", "1x", "1y", "1z", "2x", "2y", "2z"),
// u64 ranks d[3], f64 U_a (a = 0..2, column-major nmax_a x d_a), f64 core (column-major
// d1 x d2 x d3, i.e. c1 fastest); then a trailing u32 CRC-32 (IEEE 802.3, the zlib crc32) of
// every preceding byte.  Restore refuses (SVH_ECACHE) a bad magic, version, block count, tag,
// rank or CRC, a truncated file, and a cache smaller than the grid.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "internal.h"

namespace svh {

using TuckerSink = std::function<void(int q, const int* d, const std::vector<double>* U, const double* dCore,
                                      double err)>;
void tucker_hosvd_raw(svh_handle* h, double tol, const TuckerSink& sink);
void mode_products(const double* T, int Kx, int Ky, int Kz, const double* A, int hx, const double* B, int hy,
                   const double* C, int hz, double* w1, double* w2, double* out);

namespace {

constexpr uint32_t kVersion = 2;
const char* const kTags[7] = {"00", "1x", "1y", "1z", "2x", "2y", "2z"};

uint32_t crc32_update(uint32_t crc, const void* data, size_t n) {
    static uint32_t table[256];
    static bool init = false;
    if (!init) {
        for (uint32_t i = 0; i < 256; ++i) {
            uint32_t c = i;
            for (int k = 0; k < 8; ++k) c = (c & 1u) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
            table[i] = c;
        }
        init = true;
    }
    const unsigned char* p = static_cast<const unsigned char*>(data);
    crc = ~crc;
    for (size_t i = 0; i < n; ++i) crc = table[(crc ^ p[i]) & 0xFFu] ^ (crc >> 8);
    return ~crc;
}

__global__ void k_unweight(const double* __restrict__ w, double* __restrict__ t, int Kx, int Ky, int Kz) {
    const int64_t Kt = (int64_t)Kx * Ky * Kz;
    const int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (id >= Kt) return;
    const int x = (int)(id % Kx), y = (int)((id / Kx) % Ky), z = (int)(id / ((int64_t)Kx * Ky));
    t[id] = w[id] * (x ? M_SQRT1_2 : 1.0) * (y ? M_SQRT1_2 : 1.0) * (z ? M_SQRT1_2 : 1.0);
}

struct File {
    FILE* f = nullptr;
    File(const char* p, const char* m) : f(std::fopen(p, m)) {}
    ~File() {
        if (f) std::fclose(f);
    }
};

// writer that keeps the running CRC-32 of everything written
struct Writer {
    FILE* f;
    uint32_t crc = 0;
    template <typename T>
    void put(const T* v, size_t n) {
        SVH_CHECK(std::fwrite(v, sizeof(T), n, f) == n, SVH_ECACHE, "kernel cache: write failed");
        crc = crc32_update(crc, v, sizeof(T) * n);
    }
};
// reader over the whole file in memory (CRC checked before anything is parsed)
struct Reader {
    std::vector<unsigned char> buf;
    size_t pos = 0, end = 0;
    template <typename T>
    void get(T* v, size_t n) {
        SVH_CHECK(end - pos >= sizeof(T) * n, SVH_ECACHE, "kernel cache: truncated file");
        std::memcpy(v, buf.data() + pos, sizeof(T) * n);
        pos += sizeof(T) * n;
    }
};

}  // namespace

void kernel_cache_build(const char* path, const int* nmax, double tol, int device) {
    SVH_CHECK(path && nmax && tol > 0 && tol < 1, SVH_EINVAL, "kernel cache: bad args");
    for (int a = 0; a < 3; ++a) SVH_CHECK(nmax[a] >= 1 && nmax[a] <= 2048, SVH_EINVAL, "kernel cache: bad extent");
    SVH_CUDA(cudaSetDevice(device));
    // a bare handle that carries only the offset domain (compute_kernels / HOSVD use kx..kz, Kt)
    std::unique_ptr<svh_handle> h(new svh_handle());
    h->device = device;
    h->kx = nmax[0];
    h->ky = nmax[1];
    h->kz = nmax[2];
    h->Kt = (int64_t)h->kx * h->ky * h->kz;
    compute_kernels(h.get());
    File fo(path, "wb");
    SVH_CHECK(fo.f, SVH_ECACHE, std::string("kernel cache: cannot open ") + path);
    Writer w{fo.f};
    w.put("SVXT", 4);
    w.put(&kVersion, 1);
    w.put(&tol, 1);
    const uint64_t n64[3] = {(uint64_t)nmax[0], (uint64_t)nmax[1], (uint64_t)nmax[2]};
    w.put(n64, 3);
    const uint32_t nblocks = 7;
    w.put(&nblocks, 1);
    const int K3[3] = {h->kx, h->ky, h->kz};
    tucker_hosvd_raw(h.get(), tol, [&](int q, const int* d, const std::vector<double>* U, const double* dCore, double) {
        w.put(kTags[q], 2);
        const uint64_t d64[3] = {(uint64_t)d[0], (uint64_t)d[1], (uint64_t)d[2]};
        w.put(d64, 3);
        for (int a = 0; a < 3; ++a) w.put(U[a].data(), (size_t)K3[a] * d[a]);   // first d_a columns
        std::vector<double> core((size_t)d[0] * d[1] * d[2]);
        SVH_CUDA(cudaMemcpy(core.data(), dCore, core.size() * sizeof(double), cudaMemcpyDeviceToHost));
        w.put(core.data(), core.size());
    });
    const uint32_t crc = w.crc;
    SVH_CHECK(std::fwrite(&crc, 4, 1, fo.f) == 1, SVH_ECACHE, "kernel cache: write failed");
    cudaFree(h->d_kern);
    h->d_kern = nullptr;
}

// h->d_kern [7][Kt] restored from the cache (replaces compute_kernels)
void kernel_cache_restore(svh_handle* h, const char* path) {
    Reader rd;
    {
        File fi(path, "rb");
        SVH_CHECK(fi.f, SVH_ECACHE, std::string("kernel cache: cannot open ") + path);
        std::fseek(fi.f, 0, SEEK_END);
        const long n = std::ftell(fi.f);
        std::fseek(fi.f, 0, SEEK_SET);
        SVH_CHECK(n >= 48, SVH_ECACHE, "kernel cache: truncated file");
        rd.buf.resize((size_t)n);
        SVH_CHECK(std::fread(rd.buf.data(), 1, (size_t)n, fi.f) == (size_t)n, SVH_ECACHE, "kernel cache: read failed");
        rd.end = (size_t)n - 4;
    }
    char magic[4];
    uint32_t ver = 0, nblocks = 0, crc = 0;
    uint64_t n64[3];
    double tol = 0;
    rd.get(magic, 4);
    SVH_CHECK(std::memcmp(magic, "SVXT", 4) == 0, SVH_ECACHE, "kernel cache: not an SVXT file");
    rd.get(&ver, 1);
    SVH_CHECK(ver == kVersion, SVH_ECACHE, "kernel cache: version mismatch");
    std::memcpy(&crc, rd.buf.data() + rd.end, 4);
    SVH_CHECK(crc32_update(0, rd.buf.data(), rd.end) == crc, SVH_ECACHE, "kernel cache: checksum mismatch");
    rd.get(&tol, 1);
    rd.get(n64, 3);
    rd.get(&nblocks, 1);
    SVH_CHECK(nblocks == 7, SVH_ECACHE, "kernel cache: block count is not 7");
    int nmax[3];
    for (int a = 0; a < 3; ++a) {
        SVH_CHECK(n64[a] >= 1 && n64[a] <= 2048, SVH_ECACHE, "kernel cache: corrupt N_max");
        nmax[a] = (int)n64[a];
    }
    const int K3[3] = {h->kx, h->ky, h->kz};
    for (int a = 0; a < 3; ++a)
        SVH_CHECK(K3[a] <= nmax[a], SVH_ECACHE, "kernel cache smaller than the grid (Alg. 2 needs Nmax >= K)");
    const int64_t Kt = h->Kt;
    SVH_CUDA(cudaMalloc(&h->d_kern, sizeof(double) * 7 * Kt));
    double *dCore = nullptr, *w1 = nullptr, *w2 = nullptr, *dW = nullptr, *dU[3] = {};
    auto cleanup = [&] {
        cudaFree(dCore);
        cudaFree(w1);
        cudaFree(w2);
        cudaFree(dW);
        for (auto p : dU) cudaFree(p);
    };
    try {
        SVH_CUDA(cudaMalloc(&dW, Kt * sizeof(double)));
        size_t wcap = 0;
        for (int q = 0; q < 7; ++q) {
            char tag[2];
            rd.get(tag, 2);
            SVH_CHECK(std::memcmp(tag, kTags[q], 2) == 0, SVH_ECACHE, "kernel cache: unexpected block tag");
            uint64_t d64[3];
            rd.get(d64, 3);
            int d[3];
            for (int a = 0; a < 3; ++a) {
                SVH_CHECK(d64[a] >= 1 && d64[a] <= (uint64_t)nmax[a], SVH_ECACHE, "kernel cache: corrupt ranks");
                d[a] = (int)d64[a];
            }
            for (int a = 0; a < 3; ++a) {
                std::vector<double> U((size_t)nmax[a] * d[a]), Ut((size_t)K3[a] * d[a]);
                rd.get(U.data(), U.size());
                for (int j = 0; j < d[a]; ++j)   // trim: leading K_a rows of every column
                    std::memcpy(&Ut[(size_t)j * K3[a]], &U[(size_t)j * nmax[a]], K3[a] * sizeof(double));
                cudaFree(dU[a]);
                SVH_CUDA(cudaMalloc(&dU[a], Ut.size() * sizeof(double)));
                SVH_CUDA(cudaMemcpy(dU[a], Ut.data(), Ut.size() * sizeof(double), cudaMemcpyHostToDevice));
            }
            std::vector<double> core((size_t)d[0] * d[1] * d[2]);
            rd.get(core.data(), core.size());
            cudaFree(dCore);
            SVH_CUDA(cudaMalloc(&dCore, core.size() * sizeof(double)));
            SVH_CUDA(cudaMemcpy(dCore, core.data(), core.size() * sizeof(double), cudaMemcpyHostToDevice));
            // scratch of the two intermediate mode products: K1 x d2 x d3 and K1 x K2 x d3 (the cached
            // ranks may exceed a small grid's extents)
            const size_t need = std::max((size_t)h->kx * d[1] * d[2], (size_t)h->kx * h->ky * d[2]);
            if (need > wcap) {
                cudaFree(w1);
                cudaFree(w2);
                w1 = w2 = nullptr;
                SVH_CUDA(cudaMalloc(&w1, need * sizeof(double)));
                SVH_CUDA(cudaMalloc(&w2, need * sizeof(double)));
                wcap = need;
            }
            // weighted Toeplitz block = core x_i U_i[:K_i]; then remove the 1 / sqrt(2) weights
            mode_products(dCore, d[0], d[1], d[2], dU[0], h->kx, dU[1], h->ky, dU[2], h->kz, w1, w2, dW);
            SVH_LAUNCH(k_unweight, (unsigned)((Kt + 255) / 256), 256, 0, 0, dW, h->d_kern + q * Kt, h->kx, h->ky,
                       h->kz);
        }
        SVH_CUDA(cudaDeviceSynchronize());
    } catch (...) {
        cleanup();
        throw;
    }
    cleanup();
}

}  // namespace svh
