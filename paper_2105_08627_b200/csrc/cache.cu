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
// File "SVXT" v1 (little endian): char magic[4], u32 version, i32 nmax[3], f64 tol, then per
// kernel q = 0..6: i32 d[3], f64 err, f64 U_a[nmax_a][d_a] (a = 0..2, column-major nmax_a x
// d_a), f64 core[d3][d2][d1].
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

constexpr uint32_t kVersion = 1;

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

template <typename T>
void put(FILE* f, const T* v, size_t n) {
    SVH_CHECK(std::fwrite(v, sizeof(T), n, f) == n, SVH_ECACHE, "kernel cache: write failed");
}
template <typename T>
void get(FILE* f, T* v, size_t n) {
    SVH_CHECK(std::fread(v, sizeof(T), n, f) == n, SVH_ECACHE, "kernel cache: truncated file");
}

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
    put(fo.f, "SVXT", 4);
    put(fo.f, &kVersion, 1);
    put(fo.f, nmax, 3);
    put(fo.f, &tol, 1);
    const int K3[3] = {h->kx, h->ky, h->kz};
    tucker_hosvd_raw(h.get(), tol, [&](int, const int* d, const std::vector<double>* U, const double* dCore, double err) {
        put(fo.f, d, 3);
        put(fo.f, &err, 1);
        for (int a = 0; a < 3; ++a) put(fo.f, U[a].data(), (size_t)K3[a] * d[a]);   // first d_a columns
        std::vector<double> core((size_t)d[0] * d[1] * d[2]);
        SVH_CUDA(cudaMemcpy(core.data(), dCore, core.size() * sizeof(double), cudaMemcpyDeviceToHost));
        put(fo.f, core.data(), core.size());
    });
    cudaFree(h->d_kern);
    h->d_kern = nullptr;
}

// h->d_kern [7][Kt] restored from the cache (replaces compute_kernels)
void kernel_cache_restore(svh_handle* h, const char* path) {
    File fi(path, "rb");
    SVH_CHECK(fi.f, SVH_ECACHE, std::string("kernel cache: cannot open ") + path);
    char magic[4];
    uint32_t ver = 0;
    int nmax[3];
    double tol = 0;
    get(fi.f, magic, 4);
    SVH_CHECK(std::memcmp(magic, "SVXT", 4) == 0, SVH_ECACHE, "kernel cache: not an SVXT file");
    get(fi.f, &ver, 1);
    SVH_CHECK(ver == kVersion, SVH_ECACHE, "kernel cache: version mismatch");
    get(fi.f, nmax, 3);
    get(fi.f, &tol, 1);
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
            int d[3];
            double err = 0;
            get(fi.f, d, 3);
            get(fi.f, &err, 1);
            for (int a = 0; a < 3; ++a) {
                SVH_CHECK(d[a] >= 1 && d[a] <= nmax[a], SVH_ECACHE, "kernel cache: corrupt ranks");
                std::vector<double> U((size_t)nmax[a] * d[a]), Ut((size_t)K3[a] * d[a]);
                get(fi.f, U.data(), U.size());
                for (int j = 0; j < d[a]; ++j)   // trim: leading K_a rows of every column
                    std::memcpy(&Ut[(size_t)j * K3[a]], &U[(size_t)j * nmax[a]], K3[a] * sizeof(double));
                cudaFree(dU[a]);
                SVH_CUDA(cudaMalloc(&dU[a], Ut.size() * sizeof(double)));
                SVH_CUDA(cudaMemcpy(dU[a], Ut.data(), Ut.size() * sizeof(double), cudaMemcpyHostToDevice));
            }
            std::vector<double> core((size_t)d[0] * d[1] * d[2]);
            get(fi.f, core.data(), core.size());
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
