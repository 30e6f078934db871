// libsvh internal state (not part of the C-ABI).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <vector>

#include "common.cuh"

namespace svh {
struct Solve;
}

struct SvhTucker {
    // per kernel q (7): ranks d1,d2,d3; spectral factors (fp32, [h_i][d_i]); core fp32 [d3][d2][d1]
    int ranks[7][3] = {};
    float* d_factor[7][3] = {};
    float* d_core[7] = {};
    double rel_err[7] = {};
    size_t bytes = 0;
};

// per-pass profile records: 0-4 = P5 passes A..E, 5 = the whole P3s matvec (A3 + YZ + E3)
constexpr int kProfPasses = 6;

struct svh_handle {
    int device = 0;
    int kx = 0, ky = 0, kz = 0;
    double dx = 0;
    int64_t Kt = 0, K = 0, M = 0;
    int nx = 1, ny = 1, nz = 1;          // embedding extents (powers of two >= 2K-1)
    int hx = 1, hy = 1, hz = 1;          // octant extents N/2 + 1
    double freq = 0, omega = 0;
    svh_opts opts{};
    std::vector<svh_material> mats;
    std::vector<uint8_t> h_mat;          // [Kt]
    std::vector<int32_t> h_vmap;         // [Kt] packed index or -1
    std::vector<int32_t> h_vox;          // [K] flat lattice index
    // device data
    uint8_t* d_mat = nullptr;            // [Kt]
    int32_t* d_vmap = nullptr;           // [Kt]
    int32_t* d_vox = nullptr;            // [K]
    int2* d_rowinfo = nullptr;           // [Ky*Kz][W]: {occupancy bits of 32 voxels, packed index of the first}
    int rowW = 1;                        // words per row = ceil(Kx/32)
    // empty-row / empty-plane pruning of the matvec passes (zero rows of the embedded
    // current never leave HBM untouched: they are neither written nor read)
    uint32_t* d_rowmask = nullptr;       // [Kz][rowMW] bit y set <=> row (y, z) holds a voxel
    int rowMW = 1;                       // = ceil(Ky/32)
    int32_t* d_rowlist = nullptr;        // [n_rows_ne] non-empty rows z*Ky + y, ascending
    int64_t n_rows_ne = 0;
    int32_t* d_planes = nullptr;         // [nzp] non-empty z planes, ascending
    uint8_t* d_planeok = nullptr;        // [Kz] 1 <=> plane z holds a voxel
    int nzp = 0;
    uint64_t planemask = 0;              // bit z (z < 64) of d_planeok
    uint8_t* d_matp = nullptr;           // [K] material id in packed order
    double* d_kern = nullptr;            // [7][Kt] unit-voxel kernels, fp64
    float* d_spec = nullptr;             // [7][hz][hy][hx] dense octant spectra (tucker_tol == 0)
    float* d_kvt = nullptr;              // [hx][7][hz][hy] the same, kx-major (plan P3s, built on first use)
    SvhTucker tucker;
    bool use_tucker = false;
    float2* d_zloc = nullptr;            // [n_mat + 1][5] local terms z^b (index 0 unused)
    // complex128 build (opts.precision = 1, matvec64.cu): fp64 octant spectra, local terms,
    // prefactor, twiddles and the embedding workspace
    double* d_spec64 = nullptr;          // [7][hz][hy][hx]
    double2* d_zloc64 = nullptr;         // [n_mat + 1][5]
    double gscale64 = 0;
    double2* d_tw64[3] = {nullptr, nullptr, nullptr};
    double2* W64 = nullptr;
    size_t w64_bytes = 0;
    float2* d_tw[3] = {nullptr, nullptr, nullptr};  // W_N^j tables per axis
    float gscale = 0;                    // omega * mu0 * dx / (nx ny nz)
    // matvec workspace
    float2* X1 = nullptr;                // [chunk][5][kz][ky][nx]
    float2* X2 = nullptr;                // [chunk][5][kz][ny][nx]
    int ws_rhs = 0;
    // host-buffer matvec pipeline (svh_matvec_host): double-buffered device slots, copy streams
    struct HostPipe {
        size_t cap = 0;                       // RHS per slot
        float2* din[2] = {nullptr, nullptr};
        float2* dout[2] = {nullptr, nullptr};
        cudaStream_t h2d = nullptr, d2h = nullptr;
        cudaEvent_t in_ready[2] = {}, mv_done[2] = {}, out_done[2] = {};
    };
    HostPipe* pipe = nullptr;
    // matvec plan: 5 = P5, 3 = P3s; auto-tuned per chunk size (choose_plan)
    int last_plan = 5;
    std::vector<std::pair<int, int>> plan_tuned;       // (chunk RHS, plan)
    std::vector<std::pair<float, float>> plan_ms;      // (P5 ms, P3s ms) of each tuning
    // solve-side data (built lazily by svh_solve / svh_apply_system)
    svh::Solve* solve = nullptr;
    double t_setup = 0;
    // per-pass event profiling (svh_profile_enable)
    bool prof_on = false;
    struct ProfRec {
        int pass;
        cudaEvent_t a, b;
    };
    std::vector<ProfRec> prof;
    // slab-decomposed matvec: host copy of the non-empty row list and the
    // per-(P, rank) slab row lists on the device (built on first use)
    std::vector<int32_t> h_rowlist;
    struct SlabRows {
        int P, rank;
        int32_t* d = nullptr;
        int n = 0;
    };
    std::vector<SlabRows> slab_rows;
};

namespace svh {
// matvec.cu
void matvec(svh_handle* h, const float2* I, float2* CC, int nrhs, bool green_only, bool packed,
            cudaStream_t s);
void ensure_workspace(svh_handle* h, int nrhs);
void matvec_host(svh_handle* h, const float2* I_host, float2* CC_host, int nrhs, bool green_only, int chunk,
                 cudaStream_t s);
void free_host_pipe(svh_handle* h);
void slab_sizes(const svh_handle* h, int P, int64_t* out4);
void slab_forward(svh_handle* h, int rank, int P, const float2* I, float2* send, int nrhs, cudaStream_t s);
void slab_forward_p2p(svh_handle* h, int rank, int P, const float2* I, void* const* recv1_peers,
                      uint32_t* const* flag_peers, uint32_t epoch, int nrhs, cudaStream_t s);
void slab_middle_p2p(svh_handle* h, int rank, int P, const float2* recv1, void* const* recv2_peers,
                     uint32_t* const* flag_peers, uint32_t epoch, int nrhs, cudaStream_t s);
void slab_forward_compute(svh_handle* h, int rank, int P, const float2* I, int nrhs, cudaStream_t s);
void slab_middle_compute(svh_handle* h, int rank, int P, const float2* recv, int nrhs, cudaStream_t s);
void slab_middle(svh_handle* h, int rank, int P, const float2* recv, float2* send, int nrhs, cudaStream_t s);
void slab_backward(svh_handle* h, int rank, int P, const float2* recv, const float2* I, float2* CC, int nrhs,
                   bool green_only, cudaStream_t s);
// p3s.cu (plan P3s for thin grids)
bool p3s_eligible(const svh_handle* h);
void p3s_matvec(svh_handle* h, const float2* in, float2* out, float2* XT, int nr, bool green_only, bool packed,
                cudaStream_t s);
// matvec64.cu (complex128 build)
void matvec_z(svh_handle* h, const double2* I, double2* CC, int nrhs, bool green_only, cudaStream_t s);
// quad.cu
void compute_kernels(svh_handle* h);
// cache.cu (Algorithm 2)
void kernel_cache_build(const char* path, const int* nmax, double tol, int device);
void kernel_cache_restore(svh_handle* h, const char* path);
// spectra.cu
void compute_spectra(svh_handle* h);
void compute_tucker(svh_handle* h);
void free_tucker(svh_handle* h);
// solve.cu
void free_solve(svh_handle* h);
void update_local_terms(svh_handle* h);
}  // namespace svh
