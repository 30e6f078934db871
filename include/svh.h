/*
 * svh.h -- C-ABI of libsvh, the B200 (sm_100a) hot path of SuperVoxHenry
 * (arXiv 2105.08627; PAPER.md cited as P:<line>).
 *
 * The library computes, for a voxelised superconducting structure, the
 * FFT-accelerated VIE matrix-vector product CC = Z.I of Eq. 9 with
 * the two-fluid local term (Eq. 3, App. A Eq. 16-23), the saddle-system
 * operator of Eq. 7 and the preconditioned GMRES solve
 * that turns port excitations into the port impedance / inductance matrix.
 *
 * General conventions
 *  - Every entry point returns 0 on success or a negative SVH_E* code; the
 *    thread-local message of the last failure is svh_last_error().
 *  - Host pointers are read during the call only (copied); device pointers
 *    belong to the caller and must stay valid until the work queued on the
 *    given stream completes.  The handle owns every buffer it allocates.
 *  - A handle is immutable after svh_setup except through svh_set_frequency;
 *    svh_matvec / svh_apply_system may run concurrently on distinct streams
 *    only if each stream uses its own handle workspace (see svh_opts.rhs_chunk;
 *    in this version one handle serialises its workspace: do not call
 *    svh_matvec on two streams at once with the same handle).
 *  - Units: SI.  mu = mu0 = 4*pi*1e-7 H/m.  omega = 2*pi*f.
 *  - Grid: Kx x Ky x Kz voxels of edge dx.  mat_id is uint8
 *    [Kz][Ky][Kx] (x fastest); 0 = empty voxel, m >= 1 selects mats[m-1].
 *  - Non-empty voxels are numbered 0..K-1 in x-fastest lexicographic order.
 *  - Unknown vector I = [I^x; I^y; I^z; I^2D; I^3D], component-major:
 *    element (c, k) of RHS r is at ((r*5 + c)*K + k).  Complex values are
 *    interleaved (re, im) complex64 (float2) on the matvec path.
 *  - Basis normalisation (reading G1): f^x = x^/dx^2 and the PWL
 *    bases carry 1/dx^3, so I is in amperes and the incidence matrix A is
 *    dimensionless.
 *  - Nodes (M): unique face centres; ordered x-faces, then y-faces, then
 *    z-faces, each family in flat x-fastest order over its face lattice
 *    ((Kz,Ky,Kx+1), (Kz,Ky+1,Kx), (Kz+1,Ky,Kx)), keeping faces adjacent to at
 *    least one non-empty voxel.  N = 5K + M.
 */
#ifndef SVH_H
#define SVH_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* return codes */
#define SVH_OK          0
#define SVH_EINVAL     -1   /* bad dimensions / arguments; zero non-empty voxels; bad port */
#define SVH_ENOMEM     -2   /* device or host allocation failed */
#define SVH_ECUDA      -3   /* CUDA runtime / library error */
#define SVH_ENCCL      -4   /* reserved: collective error (multi-GPU layer is in Python) */
#define SVH_ENOCONV    -5   /* GMRES not converged: best iterate returned, stats flagged */
#define SVH_EOPENPORT  -6   /* |I_port| below floor (open port) */
#define SVH_ECACHE     -7   /* Toeplitz cache (Algorithm 2): unreadable, corrupt (CRC-32), wrong version or too small */

typedef struct svh_handle svh_handle;
typedef void* svh_stream;   /* a cudaStream_t (0 = legacy default stream) */

/* domain of kx*ky*kz voxels of edge dx_m metres */
typedef struct { int32_t kx, ky, kz; double dx_m; } svh_grid;

/* P:55 Eq. 3 -- two-fluid material; lambda_L_m = +INFINITY marks a normal
 * conductor (then c = 1/sigma_n, reading G5). */
typedef struct { double sigma_n_S_per_m; double lambda_L_m; } svh_material;

/* Set of voxel faces: the faces on side (-1/+1) of axis (0=x,1=y,2=z) of every
 * voxel in the half-open box [lo, hi) (x, y, z).  Faces of empty voxels are
 * ignored. */
typedef struct { int32_t axis; int32_t side; int32_t lo[3]; int32_t hi[3]; } svh_face_rect;

/* A port (reading G13): unit potential on the + faces, 0 on the - faces. */
typedef struct { int32_t n_plus; const svh_face_rect* plus; int32_t n_minus; const svh_face_rect* minus; } svh_port;

typedef struct {
    double  tucker_tol;   /* 0 = dense octant spectra; >0 = Tucker-compressed kernels (Alg. 1) */
    int32_t restart;      /* GMRES restart (50) */
    double  rre;          /* relative residual target ||b - Ax|| / ||b|| on the true residual.  P:174 uses
                             1e-8 (MATLAB double); the default here is 1e-6 because the complex64 matvec
                             is only ~3e-7 accurate (reading G16) -- smaller targets stall */
    double  inner_tol;    /* Schur-complement inner solve tolerance (1e-8) */
    int32_t inner_maxit;  /* inner PCG iteration cap */
    int32_t max_iters;    /* total GMRES iteration cap */
    int32_t rhs_chunk;    /* max RHS per internal matvec batch (workspace sizing); 0 = auto */
    int32_t verbose;      /* 0 quiet */
    const char* kernel_cache;  /* NULL: kernels by quadrature; else an SVXT file (svh_kernel_cache_build):
                                  the grid's Toeplitz tensors are restored from it (Alg. 2) */
    int32_t plan;         /* matvec plan: 5 = P5 (x | y | fused z | y | x, any grid);
                             3 = P3s (x | fused y-z-y slab on chip | x; thin grids: Nz <= 8,
                             128 <= Nx <= 1024, Ny <= 1024, y-z slab within shared memory;
                             SVH_EINVAL at the first matvec otherwise); 0 = auto: P5, or -- where
                             P3s is eligible -- whichever of the two measures faster on the first
                             product of each RHS-chunk size.  Other values -> SVH_EINVAL */
    int32_t precision;    /* matvec arithmetic: 0 = complex64 (the FFT passes; Krylov vectors are fp64);
                             1 = complex128 build: dense fp64 spectra are kept, svh_matvec_z is available and
                             svh_solve runs its operator in fp64 (tight rre, e.g. 1e-8 / 1e-10 as the paper's
                             MATLAB double); requires tucker_tol = 0, else SVH_EINVAL */
    int32_t schur_solver; /* S^-1 inside the Schur preconditioner (Eq. 13-15): 0 = AMG-preconditioned CG
                             (default); 1 = sparse-direct comparator (Table IV
                             P:251-262): METIS-reordered sparse Cholesky of S, factored once per port
                             set on the device (cuSOLVER csrchol), exact solves (inner_tol ignored) */
} svh_opts;

typedef struct {
    int32_t iterations;        /* GMRES iterations of the last port solve */
    int32_t total_iterations;  /* summed over ports */
    int32_t inner_iterations;  /* summed inner PCG iterations */
    int32_t converged;         /* 1 if every port reached rre */
    double  final_rre;         /* worst true relative residual over ports */
    double  t_setup_s, t_solve_s, t_matvec_s, t_precond_s;   /* host wall clock */
    int32_t ranks[7][3];       /* Tucker multilinear ranks per kernel (0 if dense) */
    double  compression_ratio; /* dense octant spectra bytes / Tucker bytes (P:202 CR) */
    double  t_precond_setup_s; /* setup of the Schur solver (AMG hierarchy or Cholesky factor), Table V */
    double  precond_bytes;     /* device memory of that solver (Table IV "memory") */
    int32_t schur_solver;      /* opts.schur_solver of the solve */
    int32_t amg_levels;        /* levels of the AMG hierarchy (built on the device; 0 for schur_solver 1) */
    double  amg_op_complexity; /* AMG operator complexity: sum of level nonzeros / level-0 nonzeros */
} svh_stats;

/* svh_kernel_cache_build -- Algorithm 2, install stage: Tucker-compress the 7
 * unit-voxel Toeplitz kernels on the offset domain nmax[0] x nmax[1] x nmax[2] (tolerance tol,
 * Algorithm 1) and write them to `path` (format in csrc/cache.cu).  Any grid with K_i <=
 * nmax[i] can then be set up with svh_opts.kernel_cache = path (no 6-D quadrature; restored
 * kernels carry relative error <= tol).  Errors: SVH_EINVAL, SVH_ECACHE (I/O), SVH_ECUDA. */
int svh_kernel_cache_build(const char* path, const int32_t* nmax, double tol, int32_t device);

/* Default options: tucker_tol 0 (dense spectra; P:95 uses 1e-8 when Tucker is on), restart 50,
 * rre 1e-6 (P:174 prints 1e-8; see rre above), inner_tol 1e-8, inner_maxit 200, max_iters 2000. */
void svh_default_opts(svh_opts* o);

/*
 * svh_setup -- build lattice maps, the 7 unit-voxel Galerkin kernels by
 * fp64 quadrature (App. A/B), their circulant spectra either
 * dense (octant, fp32) or Tucker-compressed (Alg. 1, Eq. 10),
 * the per-material local terms z^b (Eq. 16-23) and the incidence data.
 *   grid     : host, dims > 0, dx > 0.
 *   mat_id   : host uint8 [kz][ky][kx]; values in 0..n_mat.
 *   mats     : host array of n_mat materials (n_mat >= 1, <= 255).
 *   freq_hz  : > 0.
 *   opts     : host, may be NULL (defaults).
 *   device   : CUDA device ordinal.
 *   out      : receives the handle.
 * Errors: SVH_EINVAL (bad args / K == 0), SVH_ENOMEM, SVH_ECUDA.
 */
int svh_setup(const svh_grid* grid, const uint8_t* mat_id, const svh_material* mats, int32_t n_mat,
              double freq_hz, const svh_opts* opts, int32_t device, svh_handle** out);

/* Change omega: only z^b and the Green prefactor j*omega*mu0*dx change (kernels are f-independent). */
int svh_set_frequency(svh_handle* h, double freq_hz);

/* K = non-empty voxels, M = unique nodes; N = 5K + M. */
int svh_unknowns(const svh_handle* h, int64_t* K, int64_t* M);

/* Embedding extents Nx, Ny, Nz (powers of two >= 2K_i - 1, reading G7). */
int svh_embedding(const svh_handle* h, int32_t* n3);

/* Matvec plan geometry (for byte accounting of the pruned passes):
 * info[0] = non-empty (y, z) rows, info[1] = non-empty z planes, info[2] = Ky*Kz rows,
 * info[3] = Kz.  Rows / planes holding no voxel are zero in every embedded current
 * and are skipped by the passes (never written or read).  info: host int64[4]. */
int svh_plan_info(const svh_handle* h, int64_t* info);

/*
 * svh_matvec -- Eq. 9: CC^b = z^b I^b + IFFT{ sum_a Z^{b,a} * FFT(I^a) }, cropped
 * to the non-empty voxels.
 *   I, CC : device complex64 [nrhs][5][K] (packed voxel order); must not alias.
 *   nrhs  : >= 1.
 *   green_only : 1 = omit the z^b I^b local term (tests of the FFT part).
 *   stream: cudaStream_t.
 * Errors: SVH_EINVAL, SVH_ECUDA.  Asynchronous w.r.t. the host.
 */
int svh_matvec(svh_handle* h, const void* I, void* CC, int32_t nrhs, int32_t green_only, svh_stream stream);

/* svh_matvec_host -- svh_matvec on HOST buffers (the end-to-end call): I_host, CC_host are
 * host complex64 [nrhs][5][K] (pinned memory for copy/compute overlap; pageable works but
 * serialises).  The RHS stream through the GPU in chunks of `chunk` (0 = 4): the H2D copy of
 * the next chunk and the D2H copy of the previous one overlap the passes of the current one.
 * Returns after CC_host is complete (synchronises `stream`).  Errors as svh_matvec. */
int svh_matvec_host(svh_handle* h, const void* I_host, void* CC_host, int32_t nrhs, int32_t green_only,
                    int32_t chunk, svh_stream stream);

/* Same operator on the lattice layout: complex64 [nrhs][5][kz][ky][kx]; input
 * values at empty voxels are ignored (treated as 0); output is 0 there. */
int svh_matvec_grid(svh_handle* h, const void* I, void* CC, int32_t nrhs, int32_t green_only, svh_stream stream);

/*
 * svh_matvec_z -- the complex128 build of Eq. 9 (SURVEY 8(b) precision c128, 8(c) c.5): the same
 * operator as svh_matvec in double precision with the fp64 dense spectra (plain full-embedding
 * FFT passes; a reference / tight-solve path, not the throughput path).
 *   I, CC : device complex128 [nrhs][5][K] (packed voxel order); must not alias.
 * Errors: SVH_EINVAL (bad args, or the handle was not set up with opts.precision = 1), SVH_ENOMEM,
 * SVH_ECUDA.  Asynchronous w.r.t. the host.
 */
int svh_matvec_z(svh_handle* h, const void* I, void* CC, int32_t nrhs, int32_t green_only, svh_stream stream);

/*
 * Slab-decomposed matvec (the operator is Eq. 9 as in svh_matvec_grid,
 * P:79-83).  P ranks, each holding the same handle (replicated setup); rank r owns the
 * y-slab r*Kyl <= y < (r+1)*Kyl of every plane, Kyl = Ky/P (requires Ky % P == 0 and
 * Nx % P == 0).  One product is three calls with two all-to-alls between them, done by
 * the caller (NCCL all_to_all_single over NVLink, equal chunks):
 *   svh_slab_forward  (I_slab -> send)        pass A on the slab, packed by destination kx-slab
 *   all-to-all        (send -> recv)
 *   svh_slab_middle   (recv -> send)          passes B, C, D on kx-slab r (Nxl = Nx/P columns)
 *   all-to-all        (send -> recv)
 *   svh_slab_backward (recv, I_slab -> CC)    pass E on the slab (+ local term unless green_only)
 * I_slab, CC_slab : device complex64 [nrhs][5][Kz][Kyl][Kx] (lattice layout of the slab, zero
 *                   at empty voxels; CC is written zero there).
 * send, recv      : device complex64, nrhs * sizes[3] elements, chunk for peer p at
 *                   p * nrhs * sizes[2] (layout [p][nrhs][5][Kz][Kyl][Nxl]); caller-owned.
 * svh_slab_sizes  : sizes[0] = Kyl, [1] = Nxl, [2] = elements per peer chunk per RHS,
 *                   [3] = send/recv elements per RHS.  Errors: SVH_EINVAL (bad P / rank).
 * The calls use the handle's matvec workspace: one slab product per handle at a time.
 */
int svh_slab_sizes(const svh_handle* h, int32_t P, int64_t* sizes);
int svh_slab_forward(svh_handle* h, int32_t rank, int32_t P, const void* I_slab, void* send, int32_t nrhs,
                     svh_stream stream);
int svh_slab_middle(svh_handle* h, int32_t rank, int32_t P, const void* recv, void* send, int32_t nrhs,
                    svh_stream stream);
int svh_slab_backward(svh_handle* h, int32_t rank, int32_t P, const void* recv, const void* I_slab, void* CC_slab,
                      int32_t nrhs, int32_t green_only, svh_stream stream);

/*
 * Fused-exchange slab matvec (fused variant; operator Eq. 9): the same
 * product as svh_slab_forward / middle / backward, but the pack step stores each destination's
 * chunk directly into that peer's receive buffer over NVLink peer memory and the ranks
 * synchronise with stream memory operations (a flag write preceded by a memory barrier, and a
 * stream wait -- no SM spins), so no all-to-all call, no local send buffer and no host
 * synchronisation are involved.  Per rank, caller-owned, allocated with svh_ipc_alloc and
 * mapped into every peer with svh_ipc_open (peer arrays are indexed by rank, entry `rank` =
 * the rank's own pointer):
 *   recv1, recv2 : complex64, nrhs * sizes[3] elements each (layout as recv above)
 *   flags        : uint32 [2][P], zero-initialised (svh_ipc_alloc zeroes)
 * One product with epoch e (e = 1, 2, ... increasing by one per product on every rank):
 *   svh_slab_forward_p2p(I_slab -> peers' recv1, flags slot 0 = e)
 *   svh_slab_middle_p2p (own recv1 -> peers' recv2, flags slot 1 = e)
 *   svh_slab_backward   (own recv2, I_slab -> CC)
 * Each call returns once its work, signal and wait are enqueued on `stream` (asynchronous).
 * P <= 8.  Errors: SVH_EINVAL, SVH_ECUDA (stream memory operations unavailable, IPC failure).
 *
 * svh_ipc_alloc: cudaMalloc(bytes), zero it, write its 64-byte cudaIpcMemHandle to `handle`.
 * svh_ipc_open : map a peer's handle (cudaIpcOpenMemHandle, lazy peer access) -> *dptr.
 * svh_ipc_close / svh_ipc_free: unmap a peer mapping / free an own allocation.
 */
int svh_ipc_alloc(size_t bytes, void** dptr, void* handle);
int svh_ipc_free(void* dptr);
int svh_ipc_open(const void* handle, void** dptr);
int svh_ipc_close(void* dptr);
int svh_slab_forward_p2p(svh_handle* h, int32_t rank, int32_t P, const void* I_slab, void* const* recv1_peers,
                         uint32_t* const* flag_peers, uint32_t epoch, int32_t nrhs, svh_stream stream);
int svh_slab_middle_p2p(svh_handle* h, int32_t rank, int32_t P, const void* recv1, void* const* recv2_peers,
                        uint32_t* const* flag_peers, uint32_t epoch, int32_t nrhs, svh_stream stream);

/*
 * svh_apply_system -- Eq. 7 saddle operator (reading G12 sign convention):
 *   y_I   = Z.x_I + A^T x_Phi,   y_Phi = A x_I
 * x, y : device complex64 [nrhs][5K + M].  Errors: SVH_EINVAL, SVH_ECUDA.
 */
int svh_apply_system(svh_handle* h, const void* x, void* y, int32_t nrhs, svh_stream stream);

/*
 * svh_solve -- for each port p (reading G13): Phi = 1 on p's + faces, 0 on the
 * - faces of p and on all faces of the other ports; solve the reduced saddle
 * system with right-preconditioned FGMRES(restart) using the Schur
 * complement preconditioner of Eq. 12-15 whose S^-1 is an
 * aggregation-AMG preconditioned CG (AGMG-style); port currents give
 * Y[:,p]; Z = Y^-1, L = Im(Z)/omega, R = Re(Z).
 *   ports     : host array of n_ports ports (>= 1).
 *   Z_port    : host double[2*P*P] interleaved complex (row-major), may be NULL.
 *   L_H, R_ohm: host double[P*P] row-major, may be NULL.
 *   Y_port    : host double[2*P*P] admittance columns, may be NULL.
 *   stats     : may be NULL.
 * Errors: SVH_EINVAL (bad port), SVH_ENOCONV, SVH_EOPENPORT, SVH_ECUDA.
 */
int svh_solve(svh_handle* h, const svh_port* ports, int32_t n_ports, double* Z_port, double* L_H,
              double* R_ohm, double* Y_port, svh_stats* stats);

/* Solve only the listed port columns (0-based indices into ports), writing
 * Y columns into Y_cols (host double[2 * n_ports * n_sel], column j = port sel[j]).
 * Used by the multi-GPU layer to shard ports over ranks (one RHS per port). */
int svh_solve_columns(svh_handle* h, const svh_port* ports, int32_t n_ports, const int32_t* sel,
                      int32_t n_sel, double* Y_cols, svh_stats* stats);

/* Port post-processing (reading G13): Z = Y^-1, L = Im(Z)/omega, R = Re(Z).
 *   Y_port : host double[2*P*P] interleaved complex, row-major (Y[q][p] = current at
 *            port q for a 1 V drive of port p).  Outputs as in svh_solve (any may be NULL).
 * Errors: SVH_EINVAL, SVH_EOPENPORT (singular Y).  Host only, no device work. */
int svh_y_to_zl(const double* Y_port, int32_t P, double freq_hz, double* Z_port, double* L_H, double* R_ohm);

/* Copy the 7 unit-voxel kernels (fp64 [7][kz][ky][kx], order K0, K1x, K1y, K1z,
 * K2x, K2y, K2z; non-negative offsets) to host memory (tests / diagnostics). */
int svh_get_kernels(const svh_handle* h, double* host_out);

/* Query statistics of setup (ranks, CR, timings). */
int svh_get_stats(const svh_handle* h, svh_stats* stats);

void svh_destroy(svh_handle* h);
const char* svh_last_error(void);

/* Per-pass device-time accounting of svh_matvec: while enabled, CUDA events are
 * recorded on the caller's stream around each pass: records 0..4 = the 5 passes A..E of
 * plan P5, record 5 = one whole plan-P3s product (its 3 kernels A3, YZ, E3).
 * svh_profile_read synchronises those events and returns, per record, the summed
 * milliseconds (ms[6]) and the number of launches (launches[6]) since the last
 * reset; reset != 0 clears the record.  Both pointers may be NULL. */
int svh_profile_enable(svh_handle* h, int32_t on);
int svh_profile_read(svh_handle* h, double* ms, int64_t* launches, int32_t reset);

/* The plan (3 = P3s, 5 = P5) of the last svh_matvec chunk, and the device times of the two
 * plans measured by the last auto-selection (0 if none ran).  ms_p5 / ms_p3s may be NULL. */
int svh_matvec_plan(const svh_handle* h, int32_t* plan, float* ms_p5, float* ms_p3s);

/* Number of kernel launches issued by this library since load (instrumentation). */
int64_t svh_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* SVH_H */
