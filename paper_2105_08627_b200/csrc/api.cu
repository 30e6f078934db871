// C-ABI entry points of libsvh (include/svh.h).
#include <chrono>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "internal.h"

namespace svh {
static thread_local std::string g_err;
void set_error(const std::string& m) { g_err = m; }
int64_t& launch_counter() {
    static int64_t n = 0;
    return n;
}

constexpr double kMu0 = 4e-7 * M_PI;   // P:45, reading G4

static int next_pow2_embed(int K) {
    // smallest power of two >= 2K - 1 (reading G7)
    int n = 1;
    while (n < 2 * K - 1) n <<= 1;
    return n;
}

// z^b = c / (w_b dx), c = a + j w mu b (Eq. 16-18, 22-23); w = (1,1,1,6,2)
void update_local_terms(svh_handle* h) {
    const int nm = (int)h->mats.size();
    std::vector<float2> z((size_t)(nm + 1) * 5, make_float2(0.f, 0.f));
    std::vector<double2> z64((size_t)(nm + 1) * 5, make_double2(0.0, 0.0));
    const double w = h->omega;
    const double div[5] = {1, 1, 1, 6, 2};
    for (int m = 0; m < nm; ++m) {
        const double s0 = h->mats[m].sigma_n_S_per_m, lam = h->mats[m].lambda_L_m;
        double a, b;
        if (std::isinf(lam)) {
            a = 1.0 / s0;
            b = 0.0;
        } else {
            const double g = w * kMu0 * lam * lam;
            const double den = 1.0 + (s0 * g) * (s0 * g);
            a = s0 * g * g / den;
            b = lam * lam / den;
        }
        for (int c = 0; c < 5; ++c)
        {
            z64[(size_t)(m + 1) * 5 + c] = make_double2(a / (div[c] * h->dx), w * kMu0 * b / (div[c] * h->dx));
            z[(size_t)(m + 1) * 5 + c] = make_float2((float)z64[(size_t)(m + 1) * 5 + c].x,
                                                     (float)z64[(size_t)(m + 1) * 5 + c].y);
        }
    }
    if (!h->d_zloc) SVH_CUDA(cudaMalloc(&h->d_zloc, z.size() * sizeof(float2)));
    SVH_CUDA(cudaMemcpy(h->d_zloc, z.data(), z.size() * sizeof(float2), cudaMemcpyHostToDevice));
    h->gscale = (float)(w * kMu0 * h->dx / ((double)h->nx * h->ny * h->nz));
    h->gscale64 = w * kMu0 * h->dx / ((double)h->nx * h->ny * h->nz);
    if (h->opts.precision == 1) {
        if (!h->d_zloc64) SVH_CUDA(cudaMalloc(&h->d_zloc64, z64.size() * sizeof(double2)));
        SVH_CUDA(cudaMemcpy(h->d_zloc64, z64.data(), z64.size() * sizeof(double2), cudaMemcpyHostToDevice));
    }
}

static void make_twiddles(svh_handle* h) {
    const int N3[3] = {h->nx, h->ny, h->nz};
    for (int a = 0; a < 3; ++a) {
        std::vector<float2> t(N3[a]);
        for (int j = 0; j < N3[a]; ++j) {
            const double th = -2.0 * M_PI * j / N3[a];
            t[j] = make_float2((float)std::cos(th), (float)std::sin(th));
        }
        SVH_CUDA(cudaMalloc(&h->d_tw[a], t.size() * sizeof(float2)));
        SVH_CUDA(cudaMemcpy(h->d_tw[a], t.data(), t.size() * sizeof(float2), cudaMemcpyHostToDevice));
        if (h->opts.precision == 1) {
            std::vector<double2> t64(N3[a]);
            for (int j = 0; j < N3[a]; ++j) {
                const double th = -2.0 * M_PI * j / N3[a];
                t64[j] = make_double2(std::cos(th), std::sin(th));
            }
            SVH_CUDA(cudaMalloc(&h->d_tw64[a], t64.size() * sizeof(double2)));
            SVH_CUDA(cudaMemcpy(h->d_tw64[a], t64.data(), t64.size() * sizeof(double2), cudaMemcpyHostToDevice));
        }
    }
}

static void build_lattice(svh_handle* h) {
    const int64_t Kt = h->Kt;
    h->h_vmap.assign(Kt, -1);
    h->h_vox.clear();
    for (int64_t c = 0; c < Kt; ++c)
        if (h->h_mat[c]) {
            h->h_vmap[c] = (int32_t)h->h_vox.size();
            h->h_vox.push_back((int32_t)c);
        }
    h->K = (int64_t)h->h_vox.size();
    // unique face nodes
    int64_t M = 0;
    const int kx = h->kx, ky = h->ky, kz = h->kz;
    auto occ = [&](int x, int y, int z) {
        return x >= 0 && y >= 0 && z >= 0 && x < kx && y < ky && z < kz && h->h_mat[((int64_t)z * ky + y) * kx + x];
    };
    for (int z = 0; z < kz; ++z)
        for (int y = 0; y < ky; ++y)
            for (int x = 0; x <= kx; ++x) M += occ(x - 1, y, z) || occ(x, y, z);
    for (int z = 0; z < kz; ++z)
        for (int y = 0; y <= ky; ++y)
            for (int x = 0; x < kx; ++x) M += occ(x, y - 1, z) || occ(x, y, z);
    for (int z = 0; z <= kz; ++z)
        for (int y = 0; y < ky; ++y)
            for (int x = 0; x < kx; ++x) M += occ(x, y, z - 1) || occ(x, y, z);
    h->M = M;
    SVH_CUDA(cudaMalloc(&h->d_mat, Kt));
    SVH_CUDA(cudaMemcpy(h->d_mat, h->h_mat.data(), Kt, cudaMemcpyHostToDevice));
    SVH_CUDA(cudaMalloc(&h->d_vmap, Kt * sizeof(int32_t)));
    SVH_CUDA(cudaMemcpy(h->d_vmap, h->h_vmap.data(), Kt * sizeof(int32_t), cudaMemcpyHostToDevice));
    // row occupancy words for the gather/scatter of passes A/E
    h->rowW = (kx + 31) / 32;
    const int64_t rows = (int64_t)ky * kz;
    // one sentinel row at index `rows` (first word {0, K}): the packed segment of row r is
    // [ri[r W].y, ri[(r + 1) W].y).  matp is padded for the 4-byte cp.async of pass E.
    std::vector<int2> ri((size_t)(rows + 1) * h->rowW, make_int2(0, 0));
    std::vector<uint8_t> matp(std::max<int64_t>(1, h->K) + 16, 0);
    int64_t run = 0;   // packed index of the next occupied voxel (x-fastest order)
    for (int64_t r = 0; r < rows; ++r)
        for (int w = 0; w < h->rowW; ++w) {
            unsigned m = 0;
            const int64_t first = run;
            for (int b = 0; b < 32; ++b) {
                const int x = 32 * w + b;
                if (x >= kx) break;
                const int64_t c = r * kx + x;
                if (h->h_vmap[c] >= 0) {
                    m |= 1u << b;
                    matp[h->h_vmap[c]] = h->h_mat[c];
                    ++run;
                }
            }
            ri[(size_t)r * h->rowW + w] = make_int2((int)m, (int)first);
        }
    for (int w = 0; w < h->rowW; ++w) ri[(size_t)rows * h->rowW + w] = make_int2(0, (int)run);
    // non-empty rows / planes (pass pruning)
    h->rowMW = (ky + 31) / 32;
    std::vector<uint32_t> rm((size_t)kz * h->rowMW, 0u);
    std::vector<int32_t> rl;
    std::vector<uint8_t> pok(kz, 0);
    std::vector<int32_t> pl;
    for (int64_t r = 0; r < rows; ++r) {
        bool any = false;
        for (int w = 0; w < h->rowW && !any; ++w) any = ri[(size_t)r * h->rowW + w].x != 0;
        if (!any) continue;
        const int z = (int)(r / ky), y = (int)(r % ky);
        rm[(size_t)z * h->rowMW + y / 32] |= 1u << (y % 32);
        rl.push_back((int32_t)r);
        pok[z] = 1;
    }
    h->planemask = 0;
    for (int z = 0; z < kz; ++z)
        if (pok[z]) {
            pl.push_back(z);
            if (z < 64) h->planemask |= 1ull << z;
        }
    h->n_rows_ne = (int64_t)rl.size();
    h->h_rowlist = rl;
    h->nzp = (int)pl.size();
    SVH_CHECK(h->n_rows_ne > 0, SVH_EINVAL, "no non-empty voxel");
    SVH_CUDA(cudaMalloc(&h->d_rowmask, rm.size() * sizeof(uint32_t)));
    SVH_CUDA(cudaMemcpy(h->d_rowmask, rm.data(), rm.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
    SVH_CUDA(cudaMalloc(&h->d_rowlist, rl.size() * sizeof(int32_t)));
    SVH_CUDA(cudaMemcpy(h->d_rowlist, rl.data(), rl.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    SVH_CUDA(cudaMalloc(&h->d_planes, pl.size() * sizeof(int32_t)));
    SVH_CUDA(cudaMemcpy(h->d_planes, pl.data(), pl.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    SVH_CUDA(cudaMalloc(&h->d_planeok, pok.size()));
    SVH_CUDA(cudaMemcpy(h->d_planeok, pok.data(), pok.size(), cudaMemcpyHostToDevice));
    SVH_CUDA(cudaMalloc(&h->d_rowinfo, ri.size() * sizeof(int2)));
    SVH_CUDA(cudaMemcpy(h->d_rowinfo, ri.data(), ri.size() * sizeof(int2), cudaMemcpyHostToDevice));
    SVH_CUDA(cudaMalloc(&h->d_matp, matp.size()));
    SVH_CUDA(cudaMemcpy(h->d_matp, matp.data(), matp.size(), cudaMemcpyHostToDevice));
    SVH_CUDA(cudaMalloc(&h->d_vox, std::max<int64_t>(1, h->K) * sizeof(int32_t)));
    SVH_CUDA(cudaMemcpy(h->d_vox, h->h_vox.data(), h->K * sizeof(int32_t), cudaMemcpyHostToDevice));
}

static void destroy(svh_handle* h) {
    if (!h) return;
    for (auto& r : h->prof) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    free_solve(h);
    free_tucker(h);
    cudaFree(h->d_mat);
    cudaFree(h->d_vmap);
    cudaFree(h->d_rowinfo);
    for (auto& sr : h->slab_rows) cudaFree(sr.d);
    cudaFree(h->d_rowmask);
    cudaFree(h->d_rowlist);
    cudaFree(h->d_planes);
    cudaFree(h->d_planeok);
    cudaFree(h->d_matp);
    cudaFree(h->d_vox);
    cudaFree(h->d_kern);
    cudaFree(h->d_spec);
    cudaFree(h->d_kvt);
    cudaFree(h->d_spec64);
    cudaFree(h->d_zloc64);
    cudaFree(h->W64);
    for (int a = 0; a < 3; ++a) cudaFree(h->d_tw64[a]);
    cudaFree(h->d_zloc);
    for (int a = 0; a < 3; ++a) cudaFree(h->d_tw[a]);
    cudaFree(h->X1);
    cudaFree(h->X2);
    free_host_pipe(h);
    delete h;
}

template <typename F>
static int guarded(F&& f) {
    try {
        f();
        return SVH_OK;
    } catch (const Error& e) {
        set_error(e.msg);
        return e.code;
    } catch (const std::bad_alloc&) {
        set_error("host allocation failed");
        return SVH_ENOMEM;
    } catch (const std::exception& e) {
        set_error(e.what());
        return SVH_EINVAL;
    }
}

}  // namespace svh

using namespace svh;

extern "C" {

void svh_default_opts(svh_opts* o) {
    if (!o) return;
    std::memset(o, 0, sizeof(*o));
    o->tucker_tol = 0.0;
    o->restart = 50;
    o->rre = 1e-6;
    o->inner_tol = 1e-8;
    o->inner_maxit = 200;
    o->max_iters = 2000;
    o->rhs_chunk = 0;
    o->verbose = 0;
}

int svh_setup(const svh_grid* grid, const uint8_t* mat_id, const svh_material* mats, int32_t n_mat,
              double freq_hz, const svh_opts* opts, int32_t device, svh_handle** out) {
    return guarded([&] {
        SVH_CHECK(grid && mat_id && mats && out, SVH_EINVAL, "null argument");
        SVH_CHECK(grid->kx > 0 && grid->ky > 0 && grid->kz > 0 && grid->dx_m > 0, SVH_EINVAL, "bad grid");
        SVH_CHECK(grid->kx <= 2048 && grid->ky <= 2048 && grid->kz <= 2048, SVH_EINVAL, "grid extent > 2048");
        SVH_CHECK(n_mat >= 1 && n_mat <= 255, SVH_EINVAL, "n_mat must be in 1..255");
        SVH_CHECK(freq_hz > 0, SVH_EINVAL, "freq must be > 0");
        for (int m = 0; m < n_mat; ++m) {
            SVH_CHECK(mats[m].sigma_n_S_per_m >= 0 && mats[m].lambda_L_m > 0, SVH_EINVAL, "bad material");
            SVH_CHECK(!(std::isinf(mats[m].lambda_L_m) && mats[m].sigma_n_S_per_m <= 0), SVH_EINVAL,
                      "normal conductor needs sigma_n > 0");
        }
        svh_opts o;
        if (opts)
            o = *opts;
        else
            svh_default_opts(&o);
        // the Hessenberg column of FGMRES lives in a fixed 4096-double device scratch
        // (solve.cu: 16 + 2 (restart + 1) doubles)
        SVH_CHECK(o.restart >= 1 && o.restart <= 2039, SVH_EINVAL, "restart must be in 1..2039");
        SVH_CHECK(o.tucker_tol >= 0 && o.tucker_tol < 1, SVH_EINVAL, "tucker_tol must be in [0, 1)");
        SVH_CHECK(o.plan == 0 || o.plan == 3 || o.plan == 5, SVH_EINVAL, "matvec plan must be 0 (auto), 3 (P3s) or 5 (P5)");
        SVH_CHECK(o.precision == 0 || o.precision == 1, SVH_EINVAL, "precision must be 0 (complex64) or 1 (complex128)");
        SVH_CHECK(o.precision == 0 || o.tucker_tol == 0, SVH_EINVAL,
                  "the complex128 build uses dense spectra (tucker_tol = 0)");
        SVH_CHECK(o.schur_solver == 0 || o.schur_solver == 1, SVH_EINVAL, "schur_solver must be 0 (AMG-PCG) or 1 (sparse Cholesky)");
        auto t0 = std::chrono::steady_clock::now();
        SVH_CUDA(cudaSetDevice(device));
        svh_handle* h = new svh_handle();
        try {
            h->device = device;
            h->kx = grid->kx;
            h->ky = grid->ky;
            h->kz = grid->kz;
            h->dx = grid->dx_m;
            h->Kt = (int64_t)h->kx * h->ky * h->kz;
            h->opts = o;
            h->mats.assign(mats, mats + n_mat);
            h->h_mat.assign(mat_id, mat_id + h->Kt);
            for (int64_t c = 0; c < h->Kt; ++c)
                SVH_CHECK(h->h_mat[c] <= n_mat, SVH_EINVAL, "mat_id out of range");
            h->nx = next_pow2_embed(h->kx);
            h->ny = next_pow2_embed(h->ky);
            h->nz = next_pow2_embed(h->kz);
            h->hx = h->nx / 2 + 1;
            h->hy = h->ny / 2 + 1;
            h->hz = h->nz / 2 + 1;
            build_lattice(h);
            SVH_CHECK(h->K > 0, SVH_EINVAL, "zero non-empty voxels");
            h->freq = freq_hz;
            h->omega = 2.0 * M_PI * freq_hz;
            update_local_terms(h);
            make_twiddles(h);
            if (h->opts.kernel_cache)
                kernel_cache_restore(h, h->opts.kernel_cache);   // Algorithm 2
            else
                compute_kernels(h);
            h->opts.kernel_cache = nullptr;   // the caller's string is not kept
            if (h->opts.tucker_tol > 0) {
                h->use_tucker = true;
                compute_tucker(h);
            } else {
                compute_spectra(h);
            }
            SVH_CUDA(cudaDeviceSynchronize());
        } catch (...) {
            destroy(h);
            throw;
        }
        h->t_setup = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        *out = h;
    });
}

int svh_kernel_cache_build(const char* path, const int32_t* nmax, double tol, int32_t device) {
    return guarded([&] { kernel_cache_build(path, nmax, tol, device); });
}

int svh_set_frequency(svh_handle* h, double freq_hz) {
    return guarded([&] {
        SVH_CHECK(h && freq_hz > 0, SVH_EINVAL, "bad args");
        SVH_CUDA(cudaSetDevice(h->device));
        h->freq = freq_hz;
        h->omega = 2.0 * M_PI * freq_hz;
        update_local_terms(h);
        free_solve(h);
    });
}

int svh_unknowns(const svh_handle* h, int64_t* K, int64_t* M) {
    return guarded([&] {
        SVH_CHECK(h, SVH_EINVAL, "null handle");
        if (K) *K = h->K;
        if (M) *M = h->M;
    });
}

int svh_embedding(const svh_handle* h, int32_t* n3) {
    return guarded([&] {
        SVH_CHECK(h && n3, SVH_EINVAL, "null arg");
        n3[0] = h->nx;
        n3[1] = h->ny;
        n3[2] = h->nz;
    });
}

int svh_plan_info(const svh_handle* h, int64_t* info) {
    return guarded([&] {
        SVH_CHECK(h && info, SVH_EINVAL, "null arg");
        info[0] = h->n_rows_ne;
        info[1] = h->nzp;
        info[2] = (int64_t)h->ky * h->kz;
        info[3] = h->kz;
    });
}

int svh_slab_sizes(const svh_handle* h, int32_t P, int64_t* sizes) {
    return guarded([&] {
        SVH_CHECK(h && sizes, SVH_EINVAL, "null arg");
        slab_sizes(h, P, sizes);
    });
}

int svh_slab_forward(svh_handle* h, int32_t rank, int32_t P, const void* I_slab, void* send, int32_t nrhs,
                     svh_stream stream) {
    return guarded([&] {
        SVH_CHECK(h && I_slab && send && nrhs >= 1, SVH_EINVAL, "bad slab args");
        SVH_CUDA(cudaSetDevice(h->device));
        slab_forward(h, rank, P, (const float2*)I_slab, (float2*)send, nrhs, (cudaStream_t)stream);
    });
}

int svh_slab_middle(svh_handle* h, int32_t rank, int32_t P, const void* recv, void* send, int32_t nrhs,
                    svh_stream stream) {
    return guarded([&] {
        SVH_CHECK(h && recv && send && recv != send && nrhs >= 1, SVH_EINVAL, "bad slab args");
        SVH_CUDA(cudaSetDevice(h->device));
        slab_middle(h, rank, P, (const float2*)recv, (float2*)send, nrhs, (cudaStream_t)stream);
    });
}

int svh_slab_backward(svh_handle* h, int32_t rank, int32_t P, const void* recv, const void* I_slab, void* CC_slab,
                      int32_t nrhs, int32_t green_only, svh_stream stream) {
    return guarded([&] {
        SVH_CHECK(h && recv && I_slab && CC_slab && I_slab != CC_slab && nrhs >= 1, SVH_EINVAL, "bad slab args");
        SVH_CUDA(cudaSetDevice(h->device));
        slab_backward(h, rank, P, (const float2*)recv, (const float2*)I_slab, (float2*)CC_slab, nrhs,
                      green_only != 0, (cudaStream_t)stream);
    });
}

int svh_matvec(svh_handle* h, const void* I, void* CC, int32_t nrhs, int32_t green_only, svh_stream stream) {
    return guarded([&] {
        SVH_CHECK(h && I && CC && nrhs >= 1 && I != CC, SVH_EINVAL, "bad matvec args");
        SVH_CUDA(cudaSetDevice(h->device));
        matvec(h, (const float2*)I, (float2*)CC, nrhs, green_only != 0, true, (cudaStream_t)stream);
    });
}

int svh_matvec_host(svh_handle* h, const void* I_host, void* CC_host, int32_t nrhs, int32_t green_only,
                    int32_t chunk, svh_stream stream) {
    return guarded([&] {
        SVH_CHECK(h && I_host && CC_host && nrhs >= 1 && I_host != CC_host, SVH_EINVAL, "bad matvec args");
        SVH_CUDA(cudaSetDevice(h->device));
        matvec_host(h, (const float2*)I_host, (float2*)CC_host, nrhs, green_only != 0, chunk, (cudaStream_t)stream);
    });
}

int svh_matvec_grid(svh_handle* h, const void* I, void* CC, int32_t nrhs, int32_t green_only, svh_stream stream) {
    return guarded([&] {
        SVH_CHECK(h && I && CC && nrhs >= 1 && I != CC, SVH_EINVAL, "bad matvec args");
        SVH_CUDA(cudaSetDevice(h->device));
        matvec(h, (const float2*)I, (float2*)CC, nrhs, green_only != 0, false, (cudaStream_t)stream);
    });
}

int svh_get_kernels(const svh_handle* h, double* host_out) {
    return guarded([&] {
        SVH_CHECK(h && host_out, SVH_EINVAL, "null arg");
        SVH_CUDA(cudaSetDevice(h->device));
        SVH_CUDA(cudaMemcpy(host_out, h->d_kern, sizeof(double) * 7 * h->Kt, cudaMemcpyDeviceToHost));
    });
}

int svh_get_stats(const svh_handle* h, svh_stats* st) {
    return guarded([&] {
        SVH_CHECK(h && st, SVH_EINVAL, "null arg");
        std::memset(st, 0, sizeof(*st));
        st->t_setup_s = h->t_setup;
        if (h->use_tucker) {
            for (int q = 0; q < 7; ++q)
                for (int a = 0; a < 3; ++a) st->ranks[q][a] = h->tucker.ranks[q][a];
            const double dense = 7.0 * h->hx * h->hy * h->hz * sizeof(float);
            st->compression_ratio = h->tucker.bytes ? dense / (double)h->tucker.bytes : 0.0;
        }
    });
}

void svh_destroy(svh_handle* h) {
    if (h) {
        cudaSetDevice(h->device);
        svh::destroy(h);
    }
}

int svh_profile_enable(svh_handle* h, int32_t on) {
    return guarded([&] {
        SVH_CHECK(h, SVH_EINVAL, "null handle");
        h->prof_on = on != 0;
    });
}

int svh_profile_read(svh_handle* h, double* ms, int64_t* launches, int32_t reset) {
    return guarded([&] {
        SVH_CHECK(h, SVH_EINVAL, "null handle");
        SVH_CUDA(cudaSetDevice(h->device));
        double acc[kProfPasses] = {};
        int64_t cnt[kProfPasses] = {};
        for (auto& r : h->prof) {
            SVH_CUDA(cudaEventSynchronize(r.b));
            float t = 0.f;
            SVH_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
            acc[r.pass] += t;
            cnt[r.pass] += 1;
        }
        for (int p = 0; p < kProfPasses; ++p) {
            if (ms) ms[p] = acc[p];
            if (launches) launches[p] = cnt[p];
        }
        if (reset) {
            for (auto& r : h->prof) {
                cudaEventDestroy(r.a);
                cudaEventDestroy(r.b);
            }
            h->prof.clear();
        }
    });
}

int svh_matvec_plan(const svh_handle* h, int32_t* plan, float* ms_p5, float* ms_p3s) {
    return guarded([&] {
        SVH_CHECK(h && plan, SVH_EINVAL, "null arg");
        *plan = h->last_plan;
        if (ms_p5) *ms_p5 = h->plan_ms.empty() ? 0.f : h->plan_ms.back().first;
        if (ms_p3s) *ms_p3s = h->plan_ms.empty() ? 0.f : h->plan_ms.back().second;
    });
}

int svh_matvec_z(svh_handle* h, const void* I, void* CC, int32_t nrhs, int32_t green_only, svh_stream stream) {
    return guarded([&] {
        SVH_CHECK(h && I && CC && nrhs >= 1 && I != CC, SVH_EINVAL, "bad matvec args");
        SVH_CUDA(cudaSetDevice(h->device));
        matvec_z(h, (const double2*)I, (double2*)CC, nrhs, green_only != 0, (cudaStream_t)stream);
    });
}

const char* svh_last_error(void) { return g_err.c_str(); }

int64_t svh_launch_count(void) { return launch_counter(); }

}  // extern "C"
