// Saddle system (Eq. 7), Schur-complement preconditioner (Eq. 12-15,
// P:150-166) with an aggregation-AMG preconditioned CG for S^-1, and
// right-preconditioned FGMRES(restart) producing port admittances.
//
// Conventions (readings G12-G15):
//  * A = outward-flux incidence (M x 5K, dimensionless).  Operator:
//      y_I = Z I + A^T Phi,   y_Phi = A I          (Eq. 7 with Phi -> -Phi)
//  * Ports: Phi fixed on port faces (1 on the driven port's + faces, 0 on all
//    other port faces); KCL rows only on free nodes; a port-less conductor gets
//    one grounded node.  The iteration keeps the full [5K + M] layout: fixed
//    nodes carry an identity row and a zero right-hand side.
//  * Preconditioner (right): Q = [Y, A^T F; F A, I - F], Y = diag|Z_ii|
//    (P:154), F = diag(free).  Q^-1 [c; d]:
//        e = F A Y^-1 c - F d,  S b = e  (S = F A Y^-1 A^T F, real SPD),
//        b_fixed = d_fixed,     a = Y^-1 (c - A^T F b)
//    S^-1 by PCG with a pairwise-aggregation AMG V-cycle (re and im parts as
//    two real right-hand sides).
//  * Krylov vectors and Hessenberg in fp64; Z.I by the complex64 matvec.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <numeric>
#include <vector>

#include <mutex>

#include <cub/cub.cuh>
#include <cusolverDn.h>
#include <cusolverSp.h>
#include <cusolverSp_LOWLEVEL_PREVIEW.h>
#include <cusparse.h>

#include "internal.h"

namespace svh {

using cd = std::complex<double>;

struct CsrDev {
    int n = 0;
    int64_t nnz = 0;
    double* dinv = nullptr;   // l1-Jacobi: 1 / sum_j |a_ij|
    // ELL copy used by the SpMV-type kernels: column-major [ellw][n] (entry k of row i at
    // k*n + i, so a warp's loads of one k are coalesced); padding col = i, val = 0
    int ellw = 0;
    int* ecol = nullptr;
    double* eval = nullptr;
    int* agg = nullptr;       // fine -> coarse aggregate (except coarsest level)
    int* cmem = nullptr;      // [nc][4] members of each aggregate (-1 padded), for the
                              // deterministic (gather) restriction
    int nc = 0;
    // K-cycle vectors of this level when it is the coarse level of a Krylov-accelerated step
    double* kv1 = nullptr;
    double* kw1 = nullptr;
    double* kr2 = nullptr;
    double* kv2 = nullptr;
    double* kw2 = nullptr;
    double* vb = nullptr;     // level right-hand side (levels >= 1) [n][2]
    double* vx = nullptr;     // level solution (levels >= 1)
    double* tmp = nullptr;    // residual scratch
    double* x2 = nullptr;     // smoother ping-pong
};

struct CsrHost {
    int n = 0;
    std::vector<int> rowptr, col;
    std::vector<double> val;
};

struct Solve {
    // lattice / incidence structure (per handle)
    int64_t M = 0, K = 0;
    std::vector<int32_t> node_vox;   // [M][2]: packed voxel on the - side / + side of the face (-1 none)
    std::vector<int8_t> node_axis;   // [M]
    std::vector<int32_t> fnode;      // [K][6]: faces -x,+x,-y,+y,-z,+z
    std::vector<int32_t> face_idx[3];
    int32_t* d_node_vox = nullptr;
    int8_t* d_node_axis = nullptr;
    int32_t* d_fnode = nullptr;
    double* d_yinv = nullptr;        // [5][K]
    std::vector<double> yinv;        // host copy
    // port-dependent (fixed set): AMG hierarchy on free nodes
    std::vector<int32_t> fixed_nodes;  // sorted
    uint8_t* d_free = nullptr;       // [M] 1 = free
    int32_t* d_free_list = nullptr;  // [nf] node ids
    int32_t* d_node2free = nullptr;  // [M] free index or -1
    int nf = 0;
    std::vector<CsrDev> levels;
    double* d_cinv = nullptr;        // dense inverse of the coarsest matrix
    int ncoarse = 0;
    // work buffers
    double* wbuf[12] = {};
    size_t wsize = 0;
    double2* d_krylov = nullptr;     // V and Zp vectors
    int krylov_m = 0;
    int64_t N = 0;
    float2* c64_in = nullptr;
    float2* c64_out = nullptr;
    double2* z_out = nullptr;        // complex128 build: Z.x of apply_sys
    double* d_red = nullptr;         // reduction scratch
    int inner_its = 0;
    // PCG with device-side scalars, one CUDA graph per iteration (V-cycle included); the
    // graph is rebuilt whenever the AMG hierarchy is (port set change)
    cudaStream_t stream = nullptr;
    std::vector<std::pair<int, cudaGraphExec_t>> pcg_graphs;   // per vector-pair count NVP
    double* d_pcg = nullptr;         // [16][2 nvp_cap]: PCG scalars (k_fcg_* slot map)
    double* d_kc = nullptr;          // [levels][8][2 nvp_cap]: K-cycle scalars per level
    double* d_part = nullptr;        // deterministic-reduction partials
    size_t part_cap = 0;
    int nvp_cap = 1;                 // vector pairs (ports) the level / work buffers hold
    int pcg_cap = 0;
    double t_matvec = 0, t_precond = 0;
    bool pre_built = false;          // the preconditioner of fixed_nodes is set up
    double t_pre_setup = 0;          // its setup wall time (Table V "preconditioner setup")
    double pre_bytes = 0;            // its device memory (AMG hierarchy or Cholesky factor)
    int64_t nnz0 = 0;                // AMG level-0 nonzeros
    double op_complexity = 0;        // AMG operator complexity: sum of level nonzeros / nnz0
    // sparse-direct Schur solve (svh_opts.schur_solver = 1, the paper's Table IV
    // comparison): S(p, p) = L L^T of the METIS nested-dissection-reordered free-node Schur
    // matrix, factored and solved on the device by cuSOLVER's csrchol
    struct Chol {
        cusolverSpHandle_t sp = nullptr;
        cusparseMatDescr_t descr = nullptr;
        csrcholInfo_t info = nullptr;
        int n = 0;
        int64_t nnz = 0;
        int *rp = nullptr, *ci = nullptr, *perm = nullptr;
        double* v = nullptr;
        void* buf = nullptr;
        double *bp = nullptr, *xp = nullptr;
        size_t internal = 0, work = 0;
    } chol;
};

// ---------------------------------------------------------------------------
// kernels
namespace {

// A I (complex fp64): node r on axis a, voxel v on its - side (node = v's +a face),
// voxel u on its + side (node = u's -a face):
//   (A I)_r = [I^a_v - I^a_u] + c2(a) (I2_v + I2_u) + c3(a) (I3_v + I3_u)
//   c2 = (1/2, -1/2, 0), c3 = (1/2, 1/2, -1)   (flux table)
__device__ __forceinline__ double2 apply_A_node(const double2* __restrict__ I, int64_t K, int64_t r,
                                                const int32_t* __restrict__ node_vox,
                                                const int8_t* __restrict__ node_axis) {
    const int a = node_axis[r];
    const int v = node_vox[2 * r], u = node_vox[2 * r + 1];
    const double c2 = a == 0 ? 0.5 : (a == 1 ? -0.5 : 0.0);
    const double c3 = a == 2 ? -1.0 : 0.5;
    double2 acc = make_double2(0, 0);
    if (v >= 0) {
        const double2 p = I[a * K + v], i2 = I[3 * K + v], i3 = I[4 * K + v];
        acc.x += p.x + c2 * i2.x + c3 * i3.x;
        acc.y += p.y + c2 * i2.y + c3 * i3.y;
    }
    if (u >= 0) {
        const double2 p = I[a * K + u], i2 = I[3 * K + u], i3 = I[4 * K + u];
        acc.x += -p.x + c2 * i2.x + c3 * i3.x;
        acc.y += -p.y + c2 * i2.y + c3 * i3.y;
    }
    return acc;
}

// A^T Phi for voxel k, all 5 bases (phi may be masked by 'free')
__device__ __forceinline__ void apply_AT_voxel(const double2* __restrict__ phi, const uint8_t* __restrict__ free_,
                                               const int32_t* __restrict__ fn, double2 (&o)[5]) {
    double2 p[6];
#pragma unroll
    for (int f = 0; f < 6; ++f) {
        const int r = fn[f];
        p[f] = (r >= 0 && (!free_ || free_[r])) ? phi[r] : make_double2(0, 0);
    }
    o[0] = make_double2(p[1].x - p[0].x, p[1].y - p[0].y);
    o[1] = make_double2(p[3].x - p[2].x, p[3].y - p[2].y);
    o[2] = make_double2(p[5].x - p[4].x, p[5].y - p[4].y);
    o[3] = make_double2(0.5 * (p[0].x + p[1].x - p[2].x - p[3].x), 0.5 * (p[0].y + p[1].y - p[2].y - p[3].y));
    o[4] = make_double2(0.5 * (p[0].x + p[1].x + p[2].x + p[3].x) - (p[4].x + p[5].x),
                        0.5 * (p[0].y + p[1].y + p[2].y + p[3].y) - (p[4].y + p[5].y));
}

__global__ void k_to_c64(const double2* __restrict__ x, float2* __restrict__ y, int64_t n) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) y[i] = make_float2((float)x[i].x, (float)x[i].y);
}

// y_I = ZI (c64 result) + A^T F Phi ; y_Phi = F A I + (1 - F) Phi
// ZT = float2 (the complex64 matvec) or double2 (the complex128 build)
template <typename ZT>
__global__ void k_sys_I(const ZT* __restrict__ zi, const double2* __restrict__ x, double2* __restrict__ y,
                        const int32_t* __restrict__ fnode, const uint8_t* __restrict__ free_, int64_t K) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= K) return;
    double2 o[5];
    apply_AT_voxel(x + 5 * K, free_, fnode + 6 * k, o);
#pragma unroll
    for (int c = 0; c < 5; ++c) {
        const ZT z = zi[c * K + k];
        y[c * K + k] = make_double2((double)z.x + o[c].x, (double)z.y + o[c].y);
    }
}

__global__ void k_sys_Phi(const double2* __restrict__ x, double2* __restrict__ y, const int32_t* __restrict__ nv,
                          const int8_t* __restrict__ na, const uint8_t* __restrict__ free_, int64_t K, int64_t M) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= M) return;
    if (free_ && !free_[r]) {
        y[5 * K + r] = x[5 * K + r];
        return;
    }
    y[5 * K + r] = apply_A_node(x, K, r, nv, na);
}

// c64 variant for svh_apply_system (all nodes free)
__global__ void k_sys_c64(const float2* __restrict__ zi, const float2* __restrict__ x, float2* __restrict__ y,
                          const int32_t* __restrict__ fnode, const int32_t* __restrict__ nv,
                          const int8_t* __restrict__ na, int64_t K, int64_t M) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < K) {
        double2 p[6];
        const int32_t* fn = fnode + 6 * t;
        double2 o[5];
        double2 phi_local[6];
        for (int f = 0; f < 6; ++f) {
            const float2 v = x[5 * K + fn[f]];
            phi_local[f] = make_double2(v.x, v.y);
        }
        (void)p;
        // reuse the fp64 helper on a 6-entry local array
        int32_t idx[6] = {0, 1, 2, 3, 4, 5};
        apply_AT_voxel(phi_local, nullptr, idx, o);
        for (int c = 0; c < 5; ++c) {
            const float2 z = zi[c * K + t];
            y[c * K + t] = make_float2((float)(z.x + o[c].x), (float)(z.y + o[c].y));
        }
    } else if (t < K + M) {
        const int64_t r = t - K;
        const int a = na[r];
        const int v = nv[2 * r], u = nv[2 * r + 1];
        const double c2 = a == 0 ? 0.5 : (a == 1 ? -0.5 : 0.0);
        const double c3 = a == 2 ? -1.0 : 0.5;
        double ax = 0, ay = 0;
        if (v >= 0) {
            const float2 p = x[a * K + v], i2 = x[3 * K + v], i3 = x[4 * K + v];
            ax += p.x + c2 * i2.x + c3 * i3.x;
            ay += p.y + c2 * i2.y + c3 * i3.y;
        }
        if (u >= 0) {
            const float2 p = x[a * K + u], i2 = x[3 * K + u], i3 = x[4 * K + u];
            ax += -p.x + c2 * i2.x + c3 * i3.x;
            ay += -p.y + c2 * i2.y + c3 * i3.y;
        }
        y[5 * K + r] = make_float2((float)ax, (float)ay);
    }
}

// ---- preconditioner pieces
// t = Y^-1 c  (complex) ; e2[f] = (A t)[node] - d[node] for free nodes, split re/im -> [nf][2]
__global__ void k_pre_e(const double2* __restrict__ c, const double* __restrict__ yinv, double2* __restrict__ t,
                        int64_t n5) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n5) t[i] = make_double2(c[i].x * yinv[i], c[i].y * yinv[i]);
}
__global__ void k_pre_e2(const double2* __restrict__ t, const double2* __restrict__ d, double* __restrict__ e2,
                         const int32_t* __restrict__ free_list, const int32_t* __restrict__ nv,
                         const int8_t* __restrict__ na, int64_t K, int nf) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= nf) return;
    const int r = free_list[f];
    const double2 at = apply_A_node(t, K, r, nv, na);
    e2[2 * f] = at.x - d[r].x;
    e2[2 * f + 1] = at.y - d[r].y;
}
// batched variants: the Schur right-hand side / solution of port slot p is pair p of [nf][NVP]
__global__ void k_pre_e2V(const double2* __restrict__ t, const double2* __restrict__ d, double* __restrict__ e2,
                          const int32_t* __restrict__ free_list, const int32_t* __restrict__ nv,
                          const int8_t* __restrict__ na, int64_t K, int nf, int NVP, int p) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= nf) return;
    const int r = free_list[f];
    const double2 at = apply_A_node(t, K, r, nv, na);
    reinterpret_cast<double2*>(e2)[(int64_t)f * NVP + p] = make_double2(at.x - d[r].x, at.y - d[r].y);
}
__global__ void k_pre_bV(const double* __restrict__ b2, const double2* __restrict__ d, double2* __restrict__ outphi,
                         const int32_t* __restrict__ node2free, int64_t M, int NVP, int p) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= M) return;
    const int f = node2free[r];
    outphi[r] = f >= 0 ? reinterpret_cast<const double2*>(b2)[(int64_t)f * NVP + p] : d[r];
}
// b[node] = b2 (free) or d (fixed); stored into out Phi part
__global__ void k_pre_b(const double* __restrict__ b2, const double2* __restrict__ d, double2* __restrict__ outphi,
                        const int32_t* __restrict__ node2free, int64_t M) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= M) return;
    const int f = node2free[r];
    outphi[r] = f >= 0 ? make_double2(b2[2 * f], b2[2 * f + 1]) : d[r];
}
// a = Y^-1 (c - A^T F b)
__global__ void k_pre_a(const double2* __restrict__ c, const double2* __restrict__ bphi, const double* __restrict__ yinv,
                        double2* __restrict__ a, const int32_t* __restrict__ fnode, const uint8_t* __restrict__ free_,
                        int64_t K) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= K) return;
    double2 o[5];
    apply_AT_voxel(bphi, free_, fnode + 6 * k, o);
#pragma unroll
    for (int q = 0; q < 5; ++q) {
        const int64_t i = q * K + k;
        a[i] = make_double2((c[i].x - o[q].x) * yinv[i], (c[i].y - o[q].y) * yinv[i]);
    }
}

// ---- AMG / PCG on NV = 2*NVP real vectors stored row-major [n][NV] (pairs as double2): one
// pair per port (re, im of the Schur right-hand side); NVP = 1 is the single-port solve, NVP = B
// the batched multi-port solve (the matrix and the cycle are shared by all B ports).
// thread t -> row t / NVP, pair t % NVP (threads of a row share its ELL loads through L1)
__global__ void k_spmvV(int n, int w, const int* __restrict__ ec, const double* __restrict__ ev,
                        const double* __restrict__ x, double* __restrict__ y, int sh) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (n << sh)) return;
    const int i = t >> sh, p = t & ((1 << sh) - 1);
    const int NVP = 1 << sh;
    const double2* x2 = reinterpret_cast<const double2*>(x);
    double a0 = 0, a1 = 0;
    for (int k = 0; k < w; ++k) {
        const double v = __ldg(&ev[(int64_t)k * n + i]);
        const double2 xj = __ldg(&x2[(int64_t)__ldg(&ec[(int64_t)k * n + i]) * NVP + p]);
        a0 = fma(v, xj.x, a0);
        a1 = fma(v, xj.y, a1);
    }
    reinterpret_cast<double2*>(y)[t] = make_double2(a0, a1);
}
// l1-Jacobi sweep: xo = x + D^-1 (b - A x); x may be null (= zero initial guess)
__global__ void k_jacobiV(int n, int w, const int* __restrict__ ec, const double* __restrict__ ev,
                          const double* __restrict__ dinv, const double* __restrict__ b, const double* __restrict__ x,
                          double* __restrict__ xo, int sh) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (n << sh)) return;
    const int i = t >> sh, p = t & ((1 << sh) - 1);
    const int NVP = 1 << sh;
    const double2 bi = reinterpret_cast<const double2*>(b)[t];
    const double d = dinv[i];
    double2 o;
    if (x) {
        const double2* x2 = reinterpret_cast<const double2*>(x);
        double a0 = 0, a1 = 0;
        for (int k = 0; k < w; ++k) {
            const double v = __ldg(&ev[(int64_t)k * n + i]);
            const double2 xj = x2[(int64_t)__ldg(&ec[(int64_t)k * n + i]) * NVP + p];
            a0 = fma(v, xj.x, a0);
            a1 = fma(v, xj.y, a1);
        }
        const double2 xi = x2[t];
        o = make_double2(xi.x + d * (bi.x - a0), xi.y + d * (bi.y - a1));
    } else {
        o = make_double2(d * bi.x, d * bi.y);
    }
    reinterpret_cast<double2*>(xo)[t] = o;
}
// r = b - A x
// the first two l1-Jacobi sweeps from a zero guess in one pass: x1 = D^-1 b, x2 = x1 + D^-1 (b - A x1)
// with x1 formed on the fly at the neighbours (the same operations, in the same order, as two
// k_jacobiV launches)
__global__ void k_jacobi2V(int n, int w, const int* __restrict__ ec, const double* __restrict__ ev,
                           const double* __restrict__ dinv, const double* __restrict__ b, double* __restrict__ xo,
                           int sh) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (n << sh)) return;
    const int i = t >> sh, p = t & ((1 << sh) - 1);
    const int NVP = 1 << sh;
    const double2* b2 = reinterpret_cast<const double2*>(b);
    double a0 = 0, a1 = 0;
    for (int k = 0; k < w; ++k) {
        const double v = __ldg(&ev[(int64_t)k * n + i]);
        const int j = __ldg(&ec[(int64_t)k * n + i]);
        const double dj = __ldg(&dinv[j]);
        const double2 bj = b2[(int64_t)j * NVP + p];
        a0 = fma(v, dj * bj.x, a0);
        a1 = fma(v, dj * bj.y, a1);
    }
    const double2 bi = b2[t];
    const double d = dinv[i];
    const double2 xi = make_double2(d * bi.x, d * bi.y);
    reinterpret_cast<double2*>(xo)[t] = make_double2(xi.x + d * (bi.x - a0), xi.y + d * (bi.y - a1));
}
__global__ void k_residV(int n, int w, const int* __restrict__ ec, const double* __restrict__ ev,
                         const double* __restrict__ b, const double* __restrict__ x, double* __restrict__ r, int sh) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (n << sh)) return;
    const int i = t >> sh, p = t & ((1 << sh) - 1);
    const int NVP = 1 << sh;
    const double2* x2 = reinterpret_cast<const double2*>(x);
    double a0 = 0, a1 = 0;
    for (int k = 0; k < w; ++k) {
        const double v = __ldg(&ev[(int64_t)k * n + i]);
        const double2 xj = x2[(int64_t)__ldg(&ec[(int64_t)k * n + i]) * NVP + p];
        a0 = fma(v, xj.x, a0);
        a1 = fma(v, xj.y, a1);
    }
    const double2 bi = reinterpret_cast<const double2*>(b)[t];
    reinterpret_cast<double2*>(r)[t] = make_double2(bi.x - a0, bi.y - a1);
}
// column v of the [n][NV] layout <-> a contiguous permuted vector (sparse-direct solve):
// gather (dir 0): y[i] = x[perm[i] NV + v];  scatter (dir 1): y[perm[i] NV + v] = x[i]
__global__ void k_col_perm(const double* __restrict__ x, double* __restrict__ y, const int* __restrict__ perm, int n,
                           int NV, int v, int dir) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t o = (int64_t)__ldg(&perm[i]) * NV + v;
    if (dir == 0)
        y[i] = x[o];
    else
        y[o] = x[i];
}

__global__ void k_zero(double* __restrict__ x, int64_t n) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) x[i] = 0.0;
}
// restriction: rc[I] = sum of r[i] over the (<= 4) members i of aggregate I, in their fixed
// order (a gather, not atomics: the result is bitwise independent of scheduling and of the
// batch width)
__global__ void k_restrictG(int nc, const int* __restrict__ mem4, const double* __restrict__ r,
                            double* __restrict__ rc, int sh) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (nc << sh)) return;
    const int I = t >> sh, p = t & ((1 << sh) - 1);
    const int NVP = 1 << sh;
    const double2* r2 = reinterpret_cast<const double2*>(r);
    double a0 = 0, a1 = 0;
    for (int k = 0; k < 4; ++k) {
        const int m = mem4[4 * I + k];
        if (m < 0) break;
        const double2 v = r2[(int64_t)m * NVP + p];
        a0 += v.x;
        a1 += v.y;
    }
    reinterpret_cast<double2*>(rc)[t] = make_double2(a0, a1);
}
// prolongation: x[i] += ec[agg[i]]
__global__ void k_prolongV(int n, const int* __restrict__ agg, const double* __restrict__ ec, double* __restrict__ x,
                           int sh) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (n << sh)) return;
    const int i = t >> sh, p = t & ((1 << sh) - 1);
    const int NVP = 1 << sh;
    const int I = (agg[i] << sh) + p;
    x[2 * t] += ec[2 * I];
    x[2 * t + 1] += ec[2 * I + 1];
}
// dense coarse solve: x = Cinv b, one warp per (row, pair)
__global__ void k_denseV(int n, const double* __restrict__ Ci, const double* __restrict__ b, double* __restrict__ x,
                         int sh) {
    const int wid = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
    const int lane = threadIdx.x & 31;
    if (wid >= (n << sh)) return;
    const int row = wid >> sh, p = wid & ((1 << sh) - 1), NVP = 1 << sh;
    double a0 = 0, a1 = 0;
    for (int j = lane; j < n; j += 32) {
        const double w = Ci[(int64_t)row * n + j];
        a0 += w * b[2 * ((int64_t)j * NVP + p)];
        a1 += w * b[2 * ((int64_t)j * NVP + p) + 1];
    }
    for (int o = 16; o > 0; o >>= 1) {
        a0 += __shfl_xor_sync(0xffffffff, a0, o);
        a1 += __shfl_xor_sync(0xffffffff, a1, o);
    }
    if (lane == 0) {
        x[2 * wid] = a0;
        x[2 * wid + 1] = a1;
    }
}
// Deterministic dot products of NV = 2^(SH+1) real vectors stored [n][NV]: up to 3 pairs
// (a_d, b_d) at once.  Block b of G (G a function of n only) sums rows [b n / G, (b+1) n / G);
// thread t of the block sums rows lo + t, lo + t + 256, ... in order for every vector v (its
// row's NV values are one contiguous 8 NV-byte run: the block reads the range coalesced, each
// vector once per pair), then a fixed shuffle tree per warp and the 8 warps in order.  The
// summation order of every vector depends only on n -- not on NV, the other vectors or
// scheduling -- so a port's inner solve is bitwise the same alone or in a batch.
constexpr int kDotBlocks = 592;
constexpr int kDotThreads = 256;
template <int SH>
__global__ void __launch_bounds__(kDotThreads)
    k_ddotP(int n, int nd, const double* __restrict__ a0, const double* __restrict__ b0,
            const double* __restrict__ a1, const double* __restrict__ b1, const double* __restrict__ a2,
            const double* __restrict__ b2, double* __restrict__ part) {
    constexpr int NV = 2 << SH;
    __shared__ double red[kDotThreads / 32][NV];
    const int lo = (int)((int64_t)n * blockIdx.x / gridDim.x), hi = (int)((int64_t)n * (blockIdx.x + 1) / gridDim.x);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int d = 0; d < nd; ++d) {
        const double2* a = reinterpret_cast<const double2*>(d == 0 ? a0 : d == 1 ? a1 : a2);
        const double2* b = reinterpret_cast<const double2*>(d == 0 ? b0 : d == 1 ? b1 : b2);
        double acc[NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) acc[v] = 0.0;
        for (int i = lo + (int)threadIdx.x; i < hi; i += kDotThreads) {
#pragma unroll
            for (int v2 = 0; v2 < NV / 2; ++v2) {
                const double2 x = __ldg(&a[(int64_t)i * (NV / 2) + v2]);
                const double2 y = __ldg(&b[(int64_t)i * (NV / 2) + v2]);
                acc[2 * v2] = fma(x.x, y.x, acc[2 * v2]);
                acc[2 * v2 + 1] = fma(x.y, y.y, acc[2 * v2 + 1]);
            }
        }
#pragma unroll
        for (int v = 0; v < NV; ++v)
            for (int o = 16; o > 0; o >>= 1) acc[v] += __shfl_xor_sync(0xffffffff, acc[v], o);
        if (lane == 0)
#pragma unroll
            for (int v = 0; v < NV; ++v) red[warp][v] = acc[v];
        __syncthreads();
        if (threadIdx.x < NV) {
            double t = 0.0;
#pragma unroll
            for (int w = 0; w < kDotThreads / 32; ++w) t += red[w][threadIdx.x];
            part[((int64_t)blockIdx.x * nd + d) * NV + threadIdx.x] = t;
        }
        __syncthreads();
    }
}
// out[d * ostride + v] = sum of the block partials in a fixed order: warp w takes items (d, v)
// w, w + 4, ...; lane l sums blocks l, l + 32, ... ascending, then a fixed shuffle tree
// (independent of NV and of the other vectors, like k_ddotP)
__global__ void k_ddotF(int nb, int nd, const double* __restrict__ part, double* __restrict__ out, int ostride,
                        int sh) {
    const int NV = 2 << sh;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int t = warp; t < nd * NV; t += nw) {
        const int d = t / NV, v = t % NV;
        double acc = 0;
        for (int b = lane; b < nb; b += 32) acc += part[((int64_t)b * nd + d) * NV + v];
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffff, acc, o);
        if (lane == 0) out[d * ostride + v] = acc;
    }
}
// x += sign alpha_v y (per vector v)
__global__ void k_axpyV(int n, const double* __restrict__ alpha, int sign, const double* __restrict__ y,
                        double* __restrict__ x, int sh) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (n << (sh + 1))) return;
    x[i] += sign * alpha[i & ((2 << sh) - 1)] * y[i];
}
// p = z + beta_v p
__global__ void k_xpbyV(int n, const double* __restrict__ z, const double* __restrict__ beta,
                        double* __restrict__ p, int sh) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (n << (sh + 1))) return;
    p[i] = z[i] + beta[i & ((2 << sh) - 1)] * p[i];
}
// Flexible CG (FCG(1), the outer iteration AGMG pairs with its K-cycle: the preconditioner is a
// nonlinear, varying operator) scalars on the device, pc = Solve::d_pcg laid out [slot][NV]:
// 0 pq = p.Ap, 1 pr = p.r, 2 rr, 3 thr, 4 alpha, 5 beta, 6 zq = z.Ap, 7 done
__global__ void k_fcg_alpha(double* pc, int NV) {
    const int v = threadIdx.x;
    if (v < NV) pc[4 * NV + v] = (pc[7 * NV + v] != 0 || pc[v] == 0) ? 0.0 : pc[NV + v] / pc[v];
}
__global__ void k_fcg_check(double* pc, int NV) {
    const int v = threadIdx.x;
    if (v < NV && pc[2 * NV + v] <= pc[3 * NV + v]) pc[7 * NV + v] = 1.0;
}
__global__ void k_fcg_beta(double* pc, int NV) {
    const int v = threadIdx.x;
    if (v < NV) pc[5 * NV + v] = (pc[7 * NV + v] != 0 || pc[v] == 0) ? 0.0 : -pc[6 * NV + v] / pc[v];
}
// K-cycle (Notay-Vassilevski; AGMG): two FCG steps on the coarse level per visit.  Scalars of a
// level at kc [slot][NV]: 0 rho1 = v1.w1, 1 alpha1 = v1.rc, 2 gamma = v2.w1, 3 beta = v2.w2,
// 4 alpha2 = v2.r2.  r2 = rc - (alpha1 / rho1) w1
__global__ void k_kc_r2(int n, const double* __restrict__ rc, const double* __restrict__ w1,
                        const double* __restrict__ kc, double* __restrict__ r2, int sh) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int NV = 2 << sh;
    if (i >= n * NV) return;
    const int v = i & (NV - 1);
    const double rho1 = kc[v], a1 = kc[NV + v];
    const double c1 = rho1 != 0 ? a1 / rho1 : 0.0;
    r2[i] = rc[i] - c1 * w1[i];
}
// x_fine += P (c1 v1 + c2 v2): ec = (a1/rho1 - gamma a2/(rho1 rho2)) v1 + (a2/rho2) v2,
// rho2 = beta - gamma^2 / rho1; prolongation fused (x[i] += ec[agg[i]])
__global__ void k_kc_prolong(int n, const int* __restrict__ agg, const double* __restrict__ v1,
                             const double* __restrict__ v2, const double* __restrict__ kc, double* __restrict__ x,
                             int sh) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int NV = 2 << sh;
    if (t >= n * NV) return;
    const int i = t / NV, v = t & (NV - 1);
    const double rho1 = kc[v], a1 = kc[NV + v], gam = kc[2 * NV + v], bet = kc[3 * NV + v], a2 = kc[4 * NV + v];
    double c1 = 0, c2 = 0;
    if (rho1 != 0) {
        const double rho2 = bet - gam * gam / rho1;
        c1 = a1 / rho1;
        if (rho2 > 1e-14 * fabs(bet)) {
            c2 = a2 / rho2;
            c1 -= gam * a2 / (rho1 * rho2);
        }
    }
    const int64_t I = (int64_t)agg[i] * NV + v;
    x[t] += c1 * v1[I] + c2 * v2[I];
}
// ---- complex Krylov helpers (double2 vectors of length n)
// part[(i nblk + b)] = sum_{e in block b's grid-stride set} conj(V_i[e]) w[e], i < m; grid (nblk, m);
// k_cdots_fin sums the blocks in order (deterministic: no atomics, fixed grid)
constexpr int kCdotBlocks = 148;
__global__ void k_cdots(int64_t n, const double2* __restrict__ V, int64_t ldv, const double2* __restrict__ w,
                        double2* __restrict__ part) {
    const int i = blockIdx.y;
    const double2* v = V + i * ldv;
    double sr = 0, si = 0;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const double2 a = v[e], b = w[e];
        sr += a.x * b.x + a.y * b.y;
        si += a.x * b.y - a.y * b.x;
    }
    for (int o = 16; o > 0; o >>= 1) {
        sr += __shfl_xor_sync(0xffffffff, sr, o);
        si += __shfl_xor_sync(0xffffffff, si, o);
    }
    __shared__ double sh[2][32];
    const int wp = threadIdx.x / 32, l = threadIdx.x & 31;
    if (l == 0) {
        sh[0][wp] = sr;
        sh[1][wp] = si;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0, b = 0;
        for (int q = 0; q < (int)(blockDim.x / 32); ++q) {
            a += sh[0][q];
            b += sh[1][q];
        }
        part[(int64_t)i * gridDim.x + blockIdx.x] = make_double2(a, b);
    }
}
__global__ void k_cdots_fin(int nb, int m, const double2* __restrict__ part, double* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    double a = 0, b = 0;
    for (int k = 0; k < nb; ++k) {
        a += part[(int64_t)i * nb + k].x;
        b += part[(int64_t)i * nb + k].y;
    }
    out[2 * i] = a;
    out[2 * i + 1] = b;
}
// w -= sum_{i<m} V_i h_i   (h complex on device)
__global__ void k_cupdate(int64_t n, const double2* __restrict__ V, int64_t ldv, const double* __restrict__ h, int m,
                          double2* __restrict__ w, double sign) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n) return;
    double2 acc = w[e];
    for (int i = 0; i < m; ++i) {
        const double2 v = V[i * ldv + e];
        const double hr = h[2 * i], hi = h[2 * i + 1];
        acc.x -= sign * (v.x * hr - v.y * hi);
        acc.y -= sign * (v.x * hi + v.y * hr);
    }
    w[e] = acc;
}
// r = b - y
__global__ void k_csub(int64_t n, const double2* __restrict__ b, const double2* __restrict__ y, double2* __restrict__ r) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e < n) r[e] = make_double2(b[e].x - y[e].x, b[e].y - y[e].y);
}
__global__ void k_cscale(int64_t n, double2* __restrict__ x, double s, double2* __restrict__ y) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e < n) y[e] = make_double2(x[e].x * s, x[e].y * s);
}
__global__ void k_port_current(const double2* __restrict__ x, const int32_t* __restrict__ nodes, int n,
                               const int32_t* __restrict__ nv, const int8_t* __restrict__ na, int64_t K,
                               double* __restrict__ out) {
    double sr = 0, si = 0;
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
        const double2 f = apply_A_node(x, K, nodes[t], nv, na);
        sr -= f.x;
        si -= f.y;
    }
    for (int o = 16; o > 0; o >>= 1) {
        sr += __shfl_xor_sync(0xffffffff, sr, o);
        si += __shfl_xor_sync(0xffffffff, si, o);
    }
    __shared__ double sh[2][32];
    const int wp = threadIdx.x / 32, l = threadIdx.x & 31;
    if (l == 0) {
        sh[0][wp] = sr;
        sh[1][wp] = si;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0, b = 0;
        for (int q = 0; q < (int)(blockDim.x / 32); ++q) {
            a += sh[0][q];
            b += sh[1][q];
        }
        out[0] = a;
        out[1] = b;
    }
}
// b_I = -A^T Phi_p (Phi_p = 1 on the given nodes) ; b_Phi = 0
__global__ void k_rhs(double2* __restrict__ b, const uint8_t* __restrict__ plus_mask, const int32_t* __restrict__ fnode,
                      int64_t K, int64_t M) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < K) {
        const int32_t* fn = fnode + 6 * t;
        double2 p[6];
        for (int f = 0; f < 6; ++f) p[f] = make_double2(plus_mask[fn[f]] ? 1.0 : 0.0, 0.0);
        int32_t idx[6] = {0, 1, 2, 3, 4, 5};
        double2 o[5];
        apply_AT_voxel(p, nullptr, idx, o);
        for (int c = 0; c < 5; ++c) b[c * K + t] = make_double2(-o[c].x, -o[c].y);
    } else if (t < K + M) {
        b[5 * K + (t - K)] = make_double2(0, 0);
    }
}

inline unsigned nblk(int64_t n, int bs = 256) { return (unsigned)((n + bs - 1) / bs); }

}  // namespace

// ---------------------------------------------------------------------------
// host: structure
static void build_structure(svh_handle* h) {
    Solve* S = new Solve();
    h->solve = S;
    const int kx = h->kx, ky = h->ky, kz = h->kz;
    S->K = h->K;
    auto vox = [&](int x, int y, int z) -> int32_t {
        if (x < 0 || y < 0 || z < 0 || x >= kx || y >= ky || z >= kz) return -1;
        return h->h_vmap[((int64_t)z * ky + y) * kx + x];
    };
    int64_t next = 0;
    // face lattices: x (kz, ky, kx+1), y (kz, ky+1, kx), z (kz+1, ky, kx)
    const int fdims[3][3] = {{kx + 1, ky, kz}, {kx, ky + 1, kz}, {kx, ky, kz + 1}};
    for (int a = 0; a < 3; ++a) {
        const int fx = fdims[a][0], fy = fdims[a][1], fz = fdims[a][2];
        S->face_idx[a].assign((size_t)fx * fy * fz, -1);
        for (int z = 0; z < fz; ++z)
            for (int y = 0; y < fy; ++y)
                for (int x = 0; x < fx; ++x) {
                    const int dxm = a == 0, dym = a == 1, dzm = a == 2;
                    const int32_t vm = vox(x - dxm, y - dym, z - dzm);   // - side: its +a face
                    const int32_t vp = vox(x, y, z);                     // + side: its -a face
                    if (vm < 0 && vp < 0) continue;
                    S->face_idx[a][((size_t)z * fy + y) * fx + x] = (int32_t)next;
                    S->node_vox.push_back(vm);
                    S->node_vox.push_back(vp);
                    S->node_axis.push_back((int8_t)a);
                    ++next;
                }
    }
    S->M = next;
    SVH_CHECK(S->M == h->M, SVH_ECUDA, "node count mismatch");
    S->fnode.resize((size_t)6 * h->K);
    for (int64_t k = 0; k < h->K; ++k) {
        const int64_t c = h->h_vox[k];
        const int x = (int)(c % kx), y = (int)((c / kx) % ky), z = (int)(c / ((int64_t)kx * ky));
        for (int a = 0; a < 3; ++a) {
            const int fx = fdims[a][0], fy = fdims[a][1];
            const int xx = x + (a == 0), yy = y + (a == 1), zz = z + (a == 2);
            S->fnode[6 * k + 2 * a] = S->face_idx[a][((size_t)z * fy + y) * fx + x];
            S->fnode[6 * k + 2 * a + 1] = S->face_idx[a][((size_t)zz * fy + yy) * fx + xx];
        }
    }
    SVH_CUDA(cudaMalloc(&S->d_node_vox, S->node_vox.size() * sizeof(int32_t)));
    SVH_CUDA(cudaMemcpy(S->d_node_vox, S->node_vox.data(), S->node_vox.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    SVH_CUDA(cudaMalloc(&S->d_node_axis, S->node_axis.size()));
    SVH_CUDA(cudaMemcpy(S->d_node_axis, S->node_axis.data(), S->node_axis.size(), cudaMemcpyHostToDevice));
    SVH_CUDA(cudaMalloc(&S->d_fnode, S->fnode.size() * sizeof(int32_t)));
    SVH_CUDA(cudaMemcpy(S->d_fnode, S->fnode.data(), S->fnode.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    // Y = |Z_ii|: z^b + j w mu0 dx T^{bb}(0)
    double k0[7];
    for (int q = 0; q < 7; ++q) SVH_CUDA(cudaMemcpy(&k0[q], h->d_kern + q * h->Kt, sizeof(double), cudaMemcpyDeviceToHost));
    const double tself[5] = {k0[0], k0[0], k0[0], k0[4] + k0[5], k0[4] + k0[5] + 4.0 * k0[6]};
    const double mu0 = 4e-7 * M_PI, w = h->omega;
    const double div[5] = {1, 1, 1, 6, 2};
    S->yinv.resize((size_t)5 * h->K);
    for (int64_t k = 0; k < h->K; ++k) {
        const svh_material& m = h->mats[h->h_mat[h->h_vox[k]] - 1];
        double a, b;
        if (std::isinf(m.lambda_L_m)) {
            a = 1.0 / m.sigma_n_S_per_m;
            b = 0.0;
        } else {
            const double g = w * mu0 * m.lambda_L_m * m.lambda_L_m;
            const double den = 1.0 + (m.sigma_n_S_per_m * g) * (m.sigma_n_S_per_m * g);
            a = m.sigma_n_S_per_m * g * g / den;
            b = m.lambda_L_m * m.lambda_L_m / den;
        }
        for (int c = 0; c < 5; ++c) {
            const cd z(a / (div[c] * h->dx), w * mu0 * b / (div[c] * h->dx) + w * mu0 * h->dx * tself[c]);
            S->yinv[c * h->K + k] = 1.0 / std::abs(z);
        }
    }
    SVH_CUDA(cudaMalloc(&S->d_yinv, S->yinv.size() * sizeof(double)));
    SVH_CUDA(cudaMemcpy(S->d_yinv, S->yinv.data(), S->yinv.size() * sizeof(double), cudaMemcpyHostToDevice));
    S->N = 5 * h->K + S->M;
}

static void drop_pcg_graph(Solve* S) {
    for (auto& g : S->pcg_graphs) cudaGraphExecDestroy(g.second);
    S->pcg_graphs.clear();
}
static void free_levels(Solve* S) {
    drop_pcg_graph(S);
    for (auto& L : S->levels) {
        cudaFree(L.vb);
        cudaFree(L.vx);
        cudaFree(L.tmp);
        cudaFree(L.x2);
        cudaFree(L.dinv);
        cudaFree(L.agg);
        cudaFree(L.cmem);
        cudaFree(L.ecol);
        cudaFree(L.eval);
        for (double* k : {L.kv1, L.kw1, L.kr2, L.kv2, L.kw2}) cudaFree(k);
    }
    S->levels.clear();
    cudaFree(S->d_kc);
    S->d_kc = nullptr;
    cudaFree(S->d_cinv);
    S->d_cinv = nullptr;
    cudaFree(S->d_free);
    cudaFree(S->d_free_list);
    cudaFree(S->d_node2free);
    S->d_free = nullptr;
    S->d_free_list = nullptr;
    S->d_node2free = nullptr;
    auto& C = S->chol;
    if (C.info) cusolverSpDestroyCsrcholInfo(C.info);
    if (C.descr) cusparseDestroyMatDescr(C.descr);
    if (C.sp) cusolverSpDestroy(C.sp);
    for (void* q : {(void*)C.rp, (void*)C.ci, (void*)C.perm, (void*)C.v, C.buf, (void*)C.bp, (void*)C.xp}) cudaFree(q);
    C = Solve::Chol{};
    S->pre_built = false;
}

void free_solve(svh_handle* h) {
    Solve* S = h->solve;
    if (!S) return;
    free_levels(S);
    cudaFree(S->d_node_vox);
    cudaFree(S->d_node_axis);
    cudaFree(S->d_fnode);
    cudaFree(S->d_yinv);
    for (auto& b : S->wbuf) cudaFree(b);
    cudaFree(S->d_krylov);
    cudaFree(S->c64_in);
    cudaFree(S->c64_out);
    cudaFree(S->z_out);
    cudaFree(S->d_red);
    cudaFree(S->d_part);
    cudaFree(S->d_pcg);
    if (S->stream) cudaStreamDestroy(S->stream);
    delete S;
    h->solve = nullptr;
}

// ---------------------------------------------------------------------------
// AMG setup on the device (the paper's AGMG): the free-node Schur
// complement S = F A Y^-1 A^T F is assembled straight into the level-0 ELL, then each level is
// coarsened by double pairwise aggregation (two matching passes, aggregates of <= 4 nodes) with
// the Galerkin product P^T A P of the piecewise-constant prolongation after each pass.  Every
// step is deterministic (a function of the matrix only, no atomics in any value), so every rank
// of a sharded solve builds the bitwise-same hierarchy.
#define SVH_CUSP(call)                                                                              \
    do {                                                                                            \
        const int st__ = (int)(call);                                                               \
        if (st__ != 0) throw Error{SVH_ECUDA, std::string(#call) + " failed: status " + std::to_string(st__)}; \
    } while (0)

namespace {

// flux coefficients of the 5 bases on the 6 faces (-x,+x,-y,+y,-z,+z)
__constant__ double c_flux[5][6] = {{-1, 1, 0, 0, 0, 0},
                                    {0, 0, -1, 1, 0, 0},
                                    {0, 0, 0, 0, -1, 1},
                                    {0.5, 0.5, -0.5, -0.5, 0, 0},
                                    {0.5, 0.5, 0.5, 0.5, -1, -1}};
constexpr int kSchurW = 11;   // <= 6 faces of each of the <= 2 voxels of a face, the face itself once

// row fi of S (free node r = flist[fi]): couplings to the free faces of its <= 2 voxels,
// S_rq = sum_b flux_b(r) flux_b(q) / Y_b(k) (Eq. 13-14); ELL column-major, l1 row sums
__global__ void k_schur_ell(int nf, const int32_t* __restrict__ flist, const int32_t* __restrict__ node_vox,
                            const int32_t* __restrict__ fnode, const int32_t* __restrict__ node2free,
                            const double* __restrict__ yinv, int64_t K, int* __restrict__ ecol,
                            double* __restrict__ eval, double* __restrict__ dinv,
                            unsigned long long* __restrict__ nnz) {
    const int fi = blockIdx.x * blockDim.x + threadIdx.x;
    if (fi >= nf) return;
    const int32_t r = flist[fi];
    int cols[kSchurW];
    double vals[kSchurW];
    int cnt = 0;
    for (int side = 0; side < 2; ++side) {
        const int32_t k = node_vox[2 * r + side];
        if (k < 0) continue;
        const int32_t* fn = fnode + 6 * (int64_t)k;
        int pr = 0;
        for (int q = 0; q < 6; ++q)
            if (fn[q] == r) pr = q;
        double y[5];
        for (int b = 0; b < 5; ++b) y[b] = yinv[b * K + k];
        for (int q = 0; q < 6; ++q) {
            const int cf = node2free[fn[q]];
            if (cf < 0) continue;
            double v = 0;
            for (int b = 0; b < 5; ++b) v += c_flux[b][pr] * c_flux[b][q] * y[b];
            int j = 0;
            while (j < cnt && cols[j] != cf) ++j;
            if (j < cnt) {
                vals[j] += v;
            } else if (cnt < kSchurW) {
                cols[cnt] = cf;
                vals[cnt++] = v;
            }
        }
    }
    double s = 0;
    for (int j = 0; j < kSchurW; ++j) {
        const bool on = j < cnt;
        ecol[(int64_t)j * nf + fi] = on ? cols[j] : fi;
        eval[(int64_t)j * nf + fi] = on ? vals[j] : 0.0;
        s += on ? fabs(vals[j]) : 0.0;
    }
    dinv[fi] = s > 0 ? 1.0 / s : 0.0;
    atomicAdd(nnz, (unsigned long long)cnt);   // a count (order-independent)
}

__global__ void k_ell_diag(int n, int w, const int* __restrict__ ecol, const double* __restrict__ eval,
                           double* __restrict__ diag) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double d = 0;
    for (int k = 0; k < w; ++k)
        if (ecol[(int64_t)k * n + i] == i) d += eval[(int64_t)k * n + i];
    diag[i] = d;
}

// strength of connection (AGMG-style, negative couplings): s_ij = -a_ij / sqrt(|a_ii a_jj|)
__device__ __forceinline__ double strength(double a, double di, double dj) {
    return -a / sqrt(fabs(di * dj) + 1e-300);
}
__global__ void k_ell_smax(int n, int w, const int* __restrict__ ecol, const double* __restrict__ eval,
                           const double* __restrict__ diag, double* __restrict__ smax) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double m = 0;
    for (int k = 0; k < w; ++k) {
        const int j = ecol[(int64_t)k * n + i];
        if (j != i) m = fmax(m, strength(eval[(int64_t)k * n + i], diag[i], diag[j]));
    }
    smax[i] = m;
}

// edge tie-break: equal strengths are common on a uniform lattice; a hash of the (unordered)
// pair makes every edge key distinct, so the heaviest remaining edge is always mutually
// preferred and each matching round pairs a constant fraction of the nodes
__device__ __forceinline__ uint32_t edge_hash(uint32_t a, uint32_t b) {
    if (a > b) { const uint32_t t = a; a = b; b = t; }
    uint32_t h = a * 0x9E3779B1u ^ (b * 0x85EBCA77u + 0x7F4A7C15u);
    h ^= h >> 16; h *= 0x85EBCA6Bu; h ^= h >> 13; h *= 0xC2B2AE35u; h ^= h >> 16;
    return h;
}
// matching round, step 1: every unmatched node proposes to its strongest unmatched neighbour
// with s_ij >= 0.25 max_k s_ik (s_ij > 0); none -> it stays a singleton
__global__ void k_match_pref(int n, int w, const int* __restrict__ ecol, const double* __restrict__ eval,
                             const double* __restrict__ diag, const double* __restrict__ smax,
                             const int* __restrict__ mate, int* __restrict__ pref) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (mate[i] >= 0) {
        pref[i] = -1;
        return;
    }
    int best = -1;
    double bs = 0;
    uint32_t bh = 0;
    const double thr = 0.25 * smax[i];
    for (int k = 0; k < w; ++k) {
        const int j = ecol[(int64_t)k * n + i];
        if (j == i || mate[j] >= 0) continue;
        const double s = strength(eval[(int64_t)k * n + i], diag[i], diag[j]);
        if (!(s > 0) || s < thr) continue;
        const uint32_t hh = edge_hash(i, j);
        if (best < 0 || s > bs || (s == bs && hh > bh)) {
            best = j;
            bs = s;
            bh = hh;
        }
    }
    pref[i] = best;
}
// step 2: mutual proposals are matched; a node with no proposal is final as a singleton
__global__ void k_match_commit(int n, const int* __restrict__ pref, int* __restrict__ mate,
                               unsigned int* __restrict__ left) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || mate[i] >= 0) return;
    const int p = pref[i];
    if (p < 0)
        mate[i] = i;
    else if (pref[p] == i)
        mate[i] = p;
    else
        atomicAdd(left, 1u);   // a count only (the result does not depend on its order)
}
__global__ void k_match_final(int n, int* __restrict__ mate, int* __restrict__ lead) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (mate[i] < 0) mate[i] = i;
    lead[i] = mate[i] >= i ? 1 : 0;   // the lower node of a pair (or a singleton) opens an aggregate
}
// aggregates numbered in the order of their lowest node (keeps the spatial order of the rows)
__global__ void k_match_number(int n, const int* __restrict__ mate, const int* __restrict__ id,
                               int* __restrict__ agg, int* __restrict__ mem) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int m = mate[i];
    const int I = id[min(i, m)];
    agg[i] = I;
    if (m >= i) {
        mem[2 * I] = i;
        mem[2 * I + 1] = m > i ? m : -1;
    }
}
// Galerkin row I of P^T A P (aggregates of <= 2 nodes): the members' rows in order, columns
// mapped to aggregates, duplicates summed in first-appearance order; rows land in a [nc][2w]
// scratch, their lengths in cnt
__global__ void k_gal_rows(int nc, int n, int w, const int* __restrict__ mem, const int* __restrict__ ecol,
                           const double* __restrict__ eval, const int* __restrict__ agg, int* __restrict__ scol,
                           double* __restrict__ sval, int* __restrict__ cnt, int* __restrict__ wmax,
                           unsigned long long* __restrict__ nnz) {
    const int I = blockIdx.x * blockDim.x + threadIdx.x;
    if (I >= nc) return;
    int* rc = scol + (int64_t)I * 2 * w;
    double* rv = sval + (int64_t)I * 2 * w;
    int c = 0;
    for (int q = 0; q < 2; ++q) {
        const int m = mem[2 * I + q];
        if (m < 0) continue;
        for (int k = 0; k < w; ++k) {
            const double v = eval[(int64_t)k * n + m];
            if (v == 0.0) continue;   // ELL padding (and exact zeros)
            const int J = agg[ecol[(int64_t)k * n + m]];
            int j = 0;
            while (j < c && rc[j] != J) ++j;
            if (j < c) {
                rv[j] += v;
            } else {
                rc[c] = J;
                rv[c++] = v;
            }
        }
    }
    cnt[I] = c;
    atomicMax(wmax, c);
    atomicAdd(nnz, (unsigned long long)c);
}
__global__ void k_gal_ell(int nc, int w2, int wc, const int* __restrict__ scol, const double* __restrict__ sval,
                          const int* __restrict__ cnt, int* __restrict__ ecol, double* __restrict__ eval,
                          double* __restrict__ dinv) {
    const int I = blockIdx.x * blockDim.x + threadIdx.x;
    if (I >= nc) return;
    const int c = cnt[I];
    double s = 0;
    for (int k = 0; k < wc; ++k) {
        const bool on = k < c;
        const double v = on ? sval[(int64_t)I * w2 + k] : 0.0;
        ecol[(int64_t)k * nc + I] = on ? scol[(int64_t)I * w2 + k] : I;
        eval[(int64_t)k * nc + I] = v;
        s += fabs(v);
    }
    dinv[I] = s > 0 ? 1.0 / s : 0.0;
}
// double-pairwise composition: agg = agg2[agg1], members (<= 4, fixed width, -1 padded)
__global__ void k_compose(int n, int n2, const int* __restrict__ agg1, const int* __restrict__ agg2,
                          const int* __restrict__ mem1, const int* __restrict__ mem2, int* __restrict__ agg,
                          int* __restrict__ mem4) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) agg[t] = agg2[agg1[t]];
    if (t < n2) {
        int o = 0;
        for (int a = 0; a < 2; ++a) {
            const int c1 = mem2[2 * t + a];
            for (int b = 0; b < 2; ++b) {
                const int f = c1 >= 0 ? mem1[2 * c1 + b] : -1;
                if (f >= 0) mem4[4 * t + o++] = f;
            }
        }
        for (; o < 4; ++o) mem4[4 * t + o] = -1;
    }
}
// dense copy of a small ELL matrix (coarsest level), column-major n x n
__global__ void k_ell_dense(int n, int w, const int* __restrict__ ecol, const double* __restrict__ eval,
                            double* __restrict__ D) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int k = 0; k < w; ++k) {
        const double v = eval[(int64_t)k * n + i];
        if (v != 0.0) D[(int64_t)ecol[(int64_t)k * n + i] * n + i] += v;
    }
}
__global__ void k_eye(int n, double* __restrict__ B) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < (int64_t)n * n) B[t] = (t / n == t % n) ? 1.0 : 0.0;
}

// device scratch for one level's setup (freed on scope exit, also on a throw)
struct DevBuf {
    std::vector<void*> p;
    template <class T>
    T* get(size_t n) {
        void* q = nullptr;
        SVH_CUDA(cudaMalloc(&q, std::max<size_t>(1, n) * sizeof(T)));
        p.push_back(q);
        return (T*)q;
    }
    ~DevBuf() {
        for (void* q : p) cudaFree(q);
    }
};

// an ELL matrix on the device (level operator before its vectors are attached)
struct Ell {
    int n = 0, w = 0;
    int64_t nnz = 0;
    int* col = nullptr;
    double* val = nullptr;
    double* dinv = nullptr;
};
void free_ell(Ell& A) {
    cudaFree(A.col);
    cudaFree(A.val);
    cudaFree(A.dinv);
    A = Ell{};
}

// one pairwise matching pass on A: agg[n], mem[2 nc] (caller-allocated, nc <= n); returns nc
int pairwise_dev(const Ell& A, int* agg, int* mem, cudaStream_t s) {
    const int n = A.n;
    DevBuf B;
    double* diag = B.get<double>(n);
    double* smax = B.get<double>(n);
    int* mate = B.get<int>(n);
    int* pref = B.get<int>(n);
    int* lead = B.get<int>(n + 1);
    int* id = B.get<int>(n + 1);
    unsigned int* left = B.get<unsigned int>(1);
    const unsigned g = nblk(n);
    SVH_LAUNCH(k_ell_diag, g, 256, 0, s, n, A.w, A.col, A.val, diag);
    SVH_LAUNCH(k_ell_smax, g, 256, 0, s, n, A.w, A.col, A.val, diag, smax);
    SVH_CUDA(cudaMemsetAsync(mate, 0xff, n * sizeof(int), s));
    for (int round = 0; round < 12; ++round) {
        SVH_CUDA(cudaMemsetAsync(left, 0, sizeof(unsigned int), s));
        SVH_LAUNCH(k_match_pref, g, 256, 0, s, n, A.w, A.col, A.val, diag, smax, mate, pref);
        SVH_LAUNCH(k_match_commit, g, 256, 0, s, n, pref, mate, left);
        unsigned int h_left = 0;
        SVH_CUDA(cudaMemcpyAsync(&h_left, left, sizeof(h_left), cudaMemcpyDeviceToHost, s));
        SVH_CUDA(cudaStreamSynchronize(s));
        if (h_left == 0) break;
    }
    SVH_LAUNCH(k_match_final, g, 256, 0, s, n, mate, lead);
    size_t tb = 0;
    SVH_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, lead, id, n + 1, s));
    void* tmp = B.get<char>(tb);
    SVH_CUDA(cudaMemsetAsync(lead + n, 0, sizeof(int), s));
    SVH_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, lead, id, n + 1, s));
    int nc = 0;
    SVH_CUDA(cudaMemcpyAsync(&nc, id + n, sizeof(int), cudaMemcpyDeviceToHost, s));
    SVH_CUDA(cudaStreamSynchronize(s));
    SVH_LAUNCH(k_match_number, g, 256, 0, s, n, mate, id, agg, mem);
    return nc;
}

// C = P^T A P for the pairwise aggregates (agg, mem) of A
Ell galerkin_dev(const Ell& A, const int* agg, const int* mem, int nc, cudaStream_t s) {
    DevBuf B;
    const int w2 = 2 * A.w;
    int* scol = B.get<int>((size_t)nc * w2);
    double* sval = B.get<double>((size_t)nc * w2);
    int* cnt = B.get<int>(nc);
    int* wmax = B.get<int>(1);
    unsigned long long* nnz = B.get<unsigned long long>(1);
    SVH_CUDA(cudaMemsetAsync(wmax, 0, sizeof(int), s));
    SVH_CUDA(cudaMemsetAsync(nnz, 0, sizeof(unsigned long long), s));
    SVH_LAUNCH(k_gal_rows, nblk(nc), 256, 0, s, nc, A.n, A.w, mem, A.col, A.val, agg, scol, sval, cnt, wmax, nnz);
    int wc = 0;
    unsigned long long h_nnz = 0;
    SVH_CUDA(cudaMemcpyAsync(&wc, wmax, sizeof(int), cudaMemcpyDeviceToHost, s));
    SVH_CUDA(cudaMemcpyAsync(&h_nnz, nnz, sizeof(h_nnz), cudaMemcpyDeviceToHost, s));
    SVH_CUDA(cudaStreamSynchronize(s));
    Ell C;
    C.n = nc;
    C.w = std::max(1, wc);
    C.nnz = (int64_t)h_nnz;
    SVH_CUDA(cudaMalloc(&C.col, (size_t)C.w * std::max(1, nc) * sizeof(int)));
    SVH_CUDA(cudaMalloc(&C.val, (size_t)C.w * std::max(1, nc) * sizeof(double)));
    SVH_CUDA(cudaMalloc(&C.dinv, std::max(1, nc) * sizeof(double)));
    SVH_LAUNCH(k_gal_ell, nblk(nc), 256, 0, s, nc, w2, C.w, scol, sval, cnt, C.col, C.val, C.dinv);
    return C;
}

int g_upload_nvp = 1;   // vector pairs the level buffers are sized for (set by build_amg)
// a level of the hierarchy: takes ownership of A's arrays, attaches the cycle's vectors
CsrDev make_level(Ell& A) {
    CsrDev d;
    d.n = A.n;
    d.nnz = A.nnz;
    d.ellw = A.w;
    d.ecol = A.col;
    d.eval = A.val;
    d.dinv = A.dinv;
    A = Ell{};
    const size_t vb = (size_t)2 * std::max(1, d.n) * sizeof(double) * g_upload_nvp;
    for (double** k : {&d.vb, &d.vx, &d.tmp, &d.x2, &d.kv1, &d.kw1, &d.kr2, &d.kv2, &d.kw2})
        SVH_CUDA(cudaMalloc(k, vb));
    return d;
}

// host CSR copy of an ELL matrix (the sparse-direct comparator factors level 0 on the host side)
CsrHost ell_to_host(const Ell& A) {
    std::vector<int> ec((size_t)A.w * A.n);
    std::vector<double> ev((size_t)A.w * A.n);
    SVH_CUDA(cudaMemcpy(ec.data(), A.col, ec.size() * sizeof(int), cudaMemcpyDeviceToHost));
    SVH_CUDA(cudaMemcpy(ev.data(), A.val, ev.size() * sizeof(double), cudaMemcpyDeviceToHost));
    CsrHost H;
    H.n = A.n;
    H.rowptr.assign(A.n + 1, 0);
    for (int i = 0; i < A.n; ++i) {
        for (int k = 0; k < A.w; ++k) {
            const double v = ev[(size_t)k * A.n + i];
            if (v == 0.0) continue;
            H.col.push_back(ec[(size_t)k * A.n + i]);
            H.val.push_back(v);
        }
        H.rowptr[i + 1] = (int)H.col.size();
    }
    return H;
}

// inverse of the (small, SPD) coarsest matrix on the device: Cholesky (potrf) + potrs on I
double* dense_inverse_dev(const Ell& A, cudaStream_t s) {
    static cusolverDnHandle_t hs = nullptr;
    static std::once_flag once;
    std::call_once(once, [] { cusolverDnCreate(&hs); });
    SVH_CHECK(hs != nullptr, SVH_ECUDA, "cusolverDnCreate failed");
    const int n = A.n;
    DevBuf B;
    double* D = B.get<double>((size_t)n * n);
    int* info = B.get<int>(1);
    double* inv = nullptr;
    SVH_CUDA(cudaMalloc(&inv, (size_t)std::max(1, n) * n * sizeof(double)));
    SVH_CUDA(cudaMemsetAsync(D, 0, (size_t)n * n * sizeof(double), s));
    SVH_LAUNCH(k_ell_dense, nblk(n), 256, 0, s, n, A.w, A.col, A.val, D);
    SVH_LAUNCH(k_eye, nblk((int64_t)n * n), 256, 0, s, n, inv);
    SVH_CUSP(cusolverDnSetStream(hs, s));
    int lw = 0;
    SVH_CUSP(cusolverDnDpotrf_bufferSize(hs, CUBLAS_FILL_MODE_LOWER, n, D, n, &lw));
    double* work = B.get<double>(lw);
    SVH_CUSP(cusolverDnDpotrf(hs, CUBLAS_FILL_MODE_LOWER, n, D, n, work, lw, info));
    SVH_CUSP(cusolverDnDpotrs(hs, CUBLAS_FILL_MODE_LOWER, n, n, D, n, inv, n, info));
    int h_info = 0;
    SVH_CUDA(cudaMemcpyAsync(&h_info, info, sizeof(int), cudaMemcpyDeviceToHost, s));
    SVH_CUDA(cudaStreamSynchronize(s));
    if (h_info != 0) {
        cudaFree(inv);
        throw Error{SVH_ECUDA, "coarse Schur matrix not SPD"};
    }
    return inv;   // symmetric: row-major = column-major
}

}  // namespace

// f4 comparator: METIS nested-dissection order (host), permuted CSR, device Cholesky factor
static void build_chol(Solve* S, const CsrHost& A) {
    auto& C = S->chol;
    const int n = A.n;
    const int nnz = (int)A.col.size();
    C.n = n;
    C.nnz = nnz;
    SVH_CUSP(cusolverSpCreate(&C.sp));
    SVH_CUSP(cusparseCreateMatDescr(&C.descr));
    SVH_CUSP(cusparseSetMatType(C.descr, CUSPARSE_MATRIX_TYPE_GENERAL));
    SVH_CUSP(cusparseSetMatIndexBase(C.descr, CUSPARSE_INDEX_BASE_ZERO));
    std::vector<int> p(n), q(n);
    SVH_CUSP(cusolverSpXcsrmetisndHost(C.sp, n, nnz, C.descr, A.rowptr.data(), A.col.data(), nullptr, p.data()));
    for (int i = 0; i < n; ++i) q[p[i]] = i;
    // B = A(p, p): row i of B is row p[i] of A with columns renumbered by q, sorted
    std::vector<int> rp(n + 1, 0), ci(nnz);
    std::vector<double> v(nnz);
    std::vector<std::pair<int, double>> row;
    for (int i = 0; i < n; ++i) {
        row.clear();
        for (int k = A.rowptr[p[i]]; k < A.rowptr[p[i] + 1]; ++k) row.push_back({q[A.col[k]], A.val[k]});
        std::sort(row.begin(), row.end());
        rp[i + 1] = rp[i] + (int)row.size();
        for (size_t k = 0; k < row.size(); ++k) {
            ci[rp[i] + k] = row[k].first;
            v[rp[i] + k] = row[k].second;
        }
    }
    SVH_CUDA(cudaMalloc(&C.rp, (n + 1) * sizeof(int)));
    SVH_CUDA(cudaMalloc(&C.ci, std::max(1, nnz) * sizeof(int)));
    SVH_CUDA(cudaMalloc(&C.v, std::max(1, nnz) * sizeof(double)));
    SVH_CUDA(cudaMalloc(&C.perm, std::max(1, n) * sizeof(int)));
    SVH_CUDA(cudaMalloc(&C.bp, std::max(1, n) * sizeof(double)));
    SVH_CUDA(cudaMalloc(&C.xp, std::max(1, n) * sizeof(double)));
    SVH_CUDA(cudaMemcpy(C.rp, rp.data(), (n + 1) * sizeof(int), cudaMemcpyHostToDevice));
    SVH_CUDA(cudaMemcpy(C.ci, ci.data(), nnz * sizeof(int), cudaMemcpyHostToDevice));
    SVH_CUDA(cudaMemcpy(C.v, v.data(), nnz * sizeof(double), cudaMemcpyHostToDevice));
    SVH_CUDA(cudaMemcpy(C.perm, p.data(), n * sizeof(int), cudaMemcpyHostToDevice));
    SVH_CUSP(cusolverSpCreateCsrcholInfo(&C.info));
    SVH_CUSP(cusolverSpXcsrcholAnalysis(C.sp, n, nnz, C.descr, C.rp, C.ci, C.info));
    SVH_CUSP(cusolverSpDcsrcholBufferInfo(C.sp, n, nnz, C.descr, C.v, C.rp, C.ci, C.info, &C.internal, &C.work));
    SVH_CUDA(cudaMalloc(&C.buf, std::max<size_t>(C.work, 16)));
    SVH_CUSP(cusolverSpDcsrcholFactor(C.sp, n, nnz, C.descr, C.v, C.rp, C.ci, C.info, C.buf));
    int sing = -1;
    SVH_CUSP(cusolverSpDcsrcholZeroPivot(C.sp, C.info, 1e-300, &sing));
    SVH_CHECK(sing < 0, SVH_ECUDA, "Schur matrix not SPD (zero pivot in the sparse Cholesky)");
    SVH_CUDA(cudaDeviceSynchronize());
    S->pre_bytes = (double)C.internal + (double)C.work + (double)nnz * 12 + (double)n * 28;
}

// x = S^-1 b for the NV = 2 NVP real vectors of the [n][NV] layout, by the Cholesky factor
static void chol_solveV(Solve* S, const double* b, double* x, cudaStream_t s, int NVP) {
    auto& C = S->chol;
    const int NV = 2 * NVP;
    SVH_CUSP(cusolverSpSetStream(C.sp, s));
    for (int v = 0; v < NV; ++v) {
        SVH_LAUNCH(k_col_perm, nblk(C.n), 256, 0, s, b, C.bp, C.perm, C.n, NV, v, 0);
        SVH_CUSP(cusolverSpDcsrcholSolve(C.sp, C.n, C.bp, C.xp, C.info, C.buf));
        SVH_LAUNCH(k_col_perm, nblk(C.n), 256, 0, s, C.xp, x, C.perm, C.n, NV, v, 1);
    }
}

static void build_amg(svh_handle* h, const std::vector<int32_t>& fixed, int nvp) {
    Solve* S = h->solve;
    if (S->pre_built && fixed == S->fixed_nodes && nvp <= S->nvp_cap) return;
    free_levels(S);
    const auto tp0 = std::chrono::steady_clock::now();
    struct Done {   // setup time of whatever this call builds
        Solve* S;
        std::chrono::steady_clock::time_point t0;
        ~Done() { S->t_pre_setup = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); }
    } done{S, tp0};
    S->nvp_cap = std::max(1, nvp);
    g_upload_nvp = S->nvp_cap;
    S->fixed_nodes = fixed;
    std::vector<uint8_t> fr(S->M, 1);
    for (int32_t r : fixed) fr[r] = 0;
    // free nodes numbered in voxel order (key: the lower packed voxel index of the face, then the
    // axis), not by face family: the <= 11 couplings of a row of S are then a few positions
    // apart except across y rows / z planes, so the level-0 gathers of the PCG and the cycle
    // stay in L1/L2, and the pairwise aggregation sweeps the lattice in a spatial order
    std::vector<int32_t> node2free(S->M, -1), flist;
    {   // counting sort by key = 3 v + axis (stable in node id)
        const int64_t nk = 3 * S->K + 3;
        std::vector<int64_t> cnt(nk + 1, 0);
        std::vector<int32_t> key(S->M, -1);
        for (int64_t r = 0; r < S->M; ++r)
            if (fr[r]) {
                const int32_t a = S->node_vox[2 * r], b = S->node_vox[2 * r + 1];
                const int64_t v = a < 0 ? b : (b < 0 ? a : std::min(a, b));
                key[r] = (int32_t)(v * 3 + S->node_axis[r]);
                ++cnt[key[r] + 1];
            }
        for (int64_t k = 0; k < nk; ++k) cnt[k + 1] += cnt[k];
        flist.assign(cnt[nk], 0);
        for (int64_t r = 0; r < S->M; ++r)
            if (key[r] >= 0) flist[cnt[key[r]]++] = (int32_t)r;
        for (size_t f = 0; f < flist.size(); ++f) node2free[flist[f]] = (int32_t)f;
    }
    S->nf = (int)flist.size();
    SVH_CUDA(cudaMalloc(&S->d_free, S->M));
    SVH_CUDA(cudaMemcpy(S->d_free, fr.data(), S->M, cudaMemcpyHostToDevice));
    SVH_CUDA(cudaMalloc(&S->d_free_list, std::max<size_t>(1, flist.size()) * sizeof(int32_t)));
    SVH_CUDA(cudaMemcpy(S->d_free_list, flist.data(), flist.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    SVH_CUDA(cudaMalloc(&S->d_node2free, S->M * sizeof(int32_t)));
    SVH_CUDA(cudaMemcpy(S->d_node2free, node2free.data(), S->M * sizeof(int32_t), cudaMemcpyHostToDevice));
    S->pre_bytes = 0;
    if (S->nf == 0) {
        S->pre_built = true;
        return;
    }
    cudaStream_t s = nullptr;
    Ell A;
    A.n = S->nf;
    A.w = kSchurW;
    SVH_CUDA(cudaMalloc(&A.col, (size_t)A.w * A.n * sizeof(int)));
    SVH_CUDA(cudaMalloc(&A.val, (size_t)A.w * A.n * sizeof(double)));
    SVH_CUDA(cudaMalloc(&A.dinv, (size_t)A.n * sizeof(double)));
    {
        DevBuf B;
        unsigned long long* dn = B.get<unsigned long long>(1);
        SVH_CUDA(cudaMemsetAsync(dn, 0, sizeof(*dn), s));
        SVH_LAUNCH(k_schur_ell, nblk(A.n), 256, 0, s, A.n, S->d_free_list, S->d_node_vox, S->d_fnode,
                   S->d_node2free, S->d_yinv, S->K, A.col, A.val, A.dinv, dn);
        unsigned long long hn = 0;
        SVH_CUDA(cudaMemcpyAsync(&hn, dn, sizeof(hn), cudaMemcpyDeviceToHost, s));
        SVH_CUDA(cudaStreamSynchronize(s));
        A.nnz = (int64_t)hn;
    }
    struct EllGuard {   // frees whichever level operators are still owned here on a throw
        Ell* a[2];
        ~EllGuard() {
            for (Ell* e : a) free_ell(*e);
        }
    };
    Ell A1;
    EllGuard guard{{&A, &A1}};
    if (h->opts.schur_solver == 1) {
        build_chol(S, ell_to_host(A));
        S->pre_built = true;
        return;
    }
    S->nnz0 = A.nnz;
    S->op_complexity = 0;
    const int kCoarse = 1024;
    while (true) {
        if (A.n <= kCoarse) {
            S->d_cinv = dense_inverse_dev(A, s);
            S->ncoarse = A.n;
            S->levels.push_back(make_level(A));
            break;
        }
        DevBuf B;
        int* agg1 = B.get<int>(A.n);
        int* mem1 = B.get<int>(2 * (size_t)A.n);
        const int n1 = pairwise_dev(A, agg1, mem1, s);
        A1 = galerkin_dev(A, agg1, mem1, n1, s);
        int* agg2 = B.get<int>(n1);
        int* mem2 = B.get<int>(2 * (size_t)n1);
        const int n2 = pairwise_dev(A1, agg2, mem2, s);
        Ell C = galerkin_dev(A1, agg2, mem2, n2, s);
        free_ell(A1);
        const int n = A.n;
        CsrDev d = make_level(A);
        d.nc = n2;
        SVH_CUDA(cudaMalloc(&d.agg, n * sizeof(int)));
        SVH_CUDA(cudaMalloc(&d.cmem, 4 * (size_t)std::max(1, n2) * sizeof(int)));
        SVH_LAUNCH(k_compose, nblk(std::max(n, n2)), 256, 0, s, n, n2, agg1, agg2, mem1, mem2, d.agg, d.cmem);
        S->levels.push_back(d);
        A = C;
        if (n2 > 0.85 * n) {   // stalled coarsening: stop with a dense solve if small enough
            SVH_CHECK(A.n <= 8192, SVH_ECUDA, "AMG coarsening stalled");
        }
    }
    SVH_CUDA(cudaDeviceSynchronize());
    for (const auto& L : S->levels) S->op_complexity += (double)L.nnz;
    S->op_complexity /= std::max<double>(1.0, (double)S->nnz0);
    SVH_CUDA(cudaMalloc(&S->d_kc, S->levels.size() * 8 * 2 * (size_t)S->nvp_cap * sizeof(double)));
    SVH_CUDA(cudaMemset(S->d_kc, 0, S->levels.size() * 8 * 2 * (size_t)S->nvp_cap * sizeof(double)));
    for (const auto& L : S->levels)
        S->pre_bytes += (double)L.nnz * 12 + (double)L.ellw * L.n * 12 + (double)L.n * (4 + 8) +
                        (double)L.n * 2 * 8 * S->nvp_cap * 9;
    S->pre_bytes += (double)S->ncoarse * S->ncoarse * 8;
    S->pre_built = true;
}

// ---------------------------------------------------------------------------
// host: solver workspace and operators
static void ensure_work(svh_handle* h, int restart) {
    Solve* S = h->solve;
    const size_t need = (size_t)2 * std::max<int64_t>(S->nf, 1) * S->nvp_cap;
    if (S->wsize < need) {
        drop_pcg_graph(S);
        for (auto& b : S->wbuf) cudaFree(b);
        for (auto& b : S->wbuf) SVH_CUDA(cudaMalloc(&b, need * sizeof(double) * 1));
        S->wsize = need;
    }
    if (!S->d_red) SVH_CUDA(cudaMalloc(&S->d_red, 4096 * sizeof(double)));
    // reduction partials: k_ddotP (kDotBlocks x 3 dots x NV) and k_cdots (restart + 1 vectors x
    // kCdotBlocks complex)
    const size_t pneed = std::max((size_t)kDotBlocks * 3 * 2 * S->nvp_cap, (size_t)2 * (restart + 2) * kCdotBlocks);
    if (S->part_cap < pneed) {
        drop_pcg_graph(S);
        cudaFree(S->d_part);
        SVH_CUDA(cudaMalloc(&S->d_part, pneed * sizeof(double)));
        S->part_cap = pneed;
    }
    if (!S->c64_in) {
        SVH_CUDA(cudaMalloc(&S->c64_in, 5 * h->K * sizeof(float2)));
        SVH_CUDA(cudaMalloc(&S->c64_out, 5 * h->K * sizeof(float2)));
    }
    if (S->krylov_m < restart) {
        cudaFree(S->d_krylov);
        S->d_krylov = nullptr;
        // V: restart+1 vectors, Zp: restart vectors, plus 3 scratch (x, r, t)
        const size_t nv = (size_t)(2 * restart + 4);
        SVH_CUDA(cudaMalloc(&S->d_krylov, nv * S->N * sizeof(double2)));
        S->krylov_m = restart;
    }
}

// y = Asys x (fp64 complex, masked by the free set if given)
static void apply_sys(svh_handle* h, const double2* x, double2* y, bool masked, cudaStream_t s) {
    Solve* S = h->solve;
    const int64_t K = h->K, n5 = 5 * K;
    if (h->opts.precision == 1) {   // complex128 build: the operator in fp64 end to end
        if (!S->z_out) SVH_CUDA(cudaMalloc(&S->z_out, n5 * sizeof(double2)));
        matvec_z(h, x, S->z_out, 1, false, s);
        SVH_LAUNCH(k_sys_I<double2>, nblk(K), 256, 0, s, S->z_out, x, y, S->d_fnode, masked ? S->d_free : nullptr, K);
    } else {
        SVH_LAUNCH(k_to_c64, nblk(n5), 256, 0, s, x, S->c64_in, n5);
        matvec(h, S->c64_in, S->c64_out, 1, false, true, s);
        SVH_LAUNCH(k_sys_I<float2>, nblk(K), 256, 0, s, S->c64_out, x, y, S->d_fnode, masked ? S->d_free : nullptr, K);
    }
    SVH_LAUNCH(k_sys_Phi, nblk(S->M), 256, 0, s, x, y, S->d_node_vox, S->d_node_axis, masked ? S->d_free : nullptr, K,
               S->M);
}

// deterministic dot products (k_ddotP / k_ddotF): nd <= 3 pairs, results at out[d * ostride + v]
static void ddot(Solve* S, int n, int nd, const double* a0, const double* b0, const double* a1, const double* b1,
                 const double* a2, const double* b2, double* out, int ostride, int sh, cudaStream_t s) {
    const int nb = std::min(kDotBlocks, std::max(1, (n + 1023) / 1024));   // a function of n only
    switch (sh) {
        case 0: SVH_LAUNCH(k_ddotP<0>, nb, kDotThreads, 0, s, n, nd, a0, b0, a1, b1, a2, b2, S->d_part); break;
        case 1: SVH_LAUNCH(k_ddotP<1>, nb, kDotThreads, 0, s, n, nd, a0, b0, a1, b1, a2, b2, S->d_part); break;
        case 2: SVH_LAUNCH(k_ddotP<2>, nb, kDotThreads, 0, s, n, nd, a0, b0, a1, b1, a2, b2, S->d_part); break;
        case 3: SVH_LAUNCH(k_ddotP<3>, nb, kDotThreads, 0, s, n, nd, a0, b0, a1, b1, a2, b2, S->d_part); break;
        case 4: SVH_LAUNCH(k_ddotP<4>, nb, kDotThreads, 0, s, n, nd, a0, b0, a1, b1, a2, b2, S->d_part); break;
        default: throw Error{SVH_EINVAL, "ddot: at most 16 vector pairs"};
    }
    SVH_LAUNCH(k_ddotF, 1, 1024, 0, s, nb, nd, S->d_part, out, ostride, sh);
}

// AMG cycle on level l: x = B_l^-1 b for NVP vector pairs.  l1-Jacobi V(2,2) smoothing; the
// coarse-grid correction of the top kKLevels levels is Krylov-accelerated (K-cycle, AGMG
// P:166-168 / Notay-Vassilevski): two flexible-CG steps on the coarse system, each
// preconditioned by the next level's cycle; below, one plain recursive call (V-cycle).  The
// coarsest level is the exact dense solve.
constexpr int kKLevels = 3;
static void kcycle(Solve* S, int l, const double* b, double* x, cudaStream_t s, int NVP) {
    const int sh = __builtin_ctz(NVP);
    const int NV = 2 * NVP;
    const CsrDev& L = S->levels[l];
    const int n = L.n;
    const int64_t nt = (int64_t)n * NVP;
    const int last = (int)S->levels.size() - 1;
    if (l == last) {
        SVH_LAUNCH(k_denseV, nblk(nt, 8), 256, 0, s, n, S->d_cinv, b, x, sh);
        return;
    }
    const CsrDev& C = S->levels[l + 1];
    const int nc = L.nc;
    const int64_t nct = (int64_t)nc * NVP;
    SVH_LAUNCH(k_jacobi2V, nblk(nt), 256, 0, s, n, L.ellw, L.ecol, L.eval, L.dinv, b, L.x2, sh);
    SVH_LAUNCH(k_residV, nblk(nt), 256, 0, s, n, L.ellw, L.ecol, L.eval, b, L.x2, L.tmp, sh);
    SVH_LAUNCH(k_restrictG, nblk(nct), 256, 0, s, nc, L.cmem, L.tmp, C.vb, sh);
    if (l < kKLevels && l + 1 < last) {
        double* kc = S->d_kc + (size_t)l * 8 * NV;
        kcycle(S, l + 1, C.vb, C.kv1, s, NVP);
        SVH_LAUNCH(k_spmvV, nblk(nct), 256, 0, s, nc, C.ellw, C.ecol, C.eval, C.kv1, C.kw1, sh);
        ddot(S, nc, 2, C.kv1, C.kw1, C.kv1, C.vb, nullptr, nullptr, kc, NV, sh, s);
        SVH_LAUNCH(k_kc_r2, nblk(2 * nct), 256, 0, s, nc, C.vb, C.kw1, kc, C.kr2, sh);
        kcycle(S, l + 1, C.kr2, C.kv2, s, NVP);
        SVH_LAUNCH(k_spmvV, nblk(nct), 256, 0, s, nc, C.ellw, C.ecol, C.eval, C.kv2, C.kw2, sh);
        ddot(S, nc, 3, C.kv2, C.kw1, C.kv2, C.kw2, C.kv2, C.kr2, kc + 2 * NV, NV, sh, s);
        SVH_LAUNCH(k_kc_prolong, nblk(2 * nt), 256, 0, s, n, L.agg, C.kv1, C.kv2, kc, L.x2, sh);
    } else {
        kcycle(S, l + 1, C.vb, C.vx, s, NVP);
        SVH_LAUNCH(k_prolongV, nblk(nt), 256, 0, s, n, L.agg, C.vx, L.x2, sh);
    }
    // post-smoothing: L.x2 -> L.tmp (free since the restriction) -> x
    SVH_LAUNCH(k_jacobiV, nblk(nt), 256, 0, s, n, L.ellw, L.ecol, L.eval, L.dinv, b, L.x2, L.tmp, sh);
    SVH_LAUNCH(k_jacobiV, nblk(nt), 256, 0, s, n, L.ellw, L.ecol, L.eval, L.dinv, b, L.tmp, x, sh);
}

// Flexible CG (FCG(1)) on S (level 0) for NV = 2 NVP real right-hand sides (re / im of NVP
// ports), preconditioned by the K-cycle: x = S^-1 b to relative tol per vector (P:166 AGMG-CG;
// G15).  All scalars stay on the device; one iteration (SpMV, 4 deterministic dots, scalar
// updates and the whole cycle) is a CUDA graph captured once per hierarchy and NVP and replayed;
// the host reads the convergence flags every kCheck iterations.  Vectors that converge freeze
// (alpha = 0), and every reduction has a batch-independent order, so a port's result is
// bitwise the same whichever ports share its batch (1-GPU vs sharded L bit for bit).
static int pcgV(svh_handle* h, const double* b, double* x, double tol, int maxit, cudaStream_t s, int NVP) {
    Solve* S = h->solve;
    const CsrDev& A = S->levels[0];
    const int n = A.n;
    const int NV = 2 * NVP;
    const int sh = __builtin_ctz(NVP);
    SVH_CHECK((NVP & (NVP - 1)) == 0 && NVP <= 16, SVH_EINVAL, "pcg: vector pairs must be a power of two <= 16");
    const int64_t nt = (int64_t)n * NVP, nd = 2 * nt;
    double* r = S->wbuf[0];
    double* z = S->wbuf[1];
    double* p = S->wbuf[2];
    double* q = S->wbuf[3];
    double* pc = S->d_pcg;
    auto iteration = [&] {
        SVH_LAUNCH(k_spmvV, nblk(nt), 256, 0, s, n, A.ellw, A.ecol, A.eval, p, q, sh);
        ddot(S, n, 2, p, q, p, r, nullptr, nullptr, pc, NV, sh, s);   // pq, pr
        SVH_LAUNCH(k_fcg_alpha, 1, 64, 0, s, pc, NV);
        SVH_LAUNCH(k_axpyV, nblk(nd), 256, 0, s, n, pc + 4 * NV, +1, p, x, sh);
        SVH_LAUNCH(k_axpyV, nblk(nd), 256, 0, s, n, pc + 4 * NV, -1, q, r, sh);
        ddot(S, n, 1, r, r, nullptr, nullptr, nullptr, nullptr, pc + 2 * NV, NV, sh, s);
        SVH_LAUNCH(k_fcg_check, 1, 64, 0, s, pc, NV);
        kcycle(S, 0, r, z, s, NVP);
        ddot(S, n, 1, z, q, nullptr, nullptr, nullptr, nullptr, pc + 6 * NV, NV, sh, s);
        SVH_LAUNCH(k_fcg_beta, 1, 64, 0, s, pc, NV);
        SVH_LAUNCH(k_xpbyV, nblk(nd), 256, 0, s, n, z, pc + 5 * NV, p, sh);
    };
    // b.b -> thresholds thr = tol^2 b.b; vectors with b = 0 are done from the start
    ddot(S, n, 1, b, b, nullptr, nullptr, nullptr, nullptr, pc + 2 * NV, NV, sh, s);
    std::vector<double> bn(NV);
    SVH_CUDA(cudaMemcpyAsync(bn.data(), pc + 2 * NV, NV * sizeof(double), cudaMemcpyDeviceToHost, s));
    SVH_CUDA(cudaStreamSynchronize(s));
    SVH_LAUNCH(k_zero, nblk(nd), 256, 0, s, x, nd);
    bool any = false;
    std::vector<double> init(8 * NV, 0.0);
    for (int v = 0; v < NV; ++v) {
        init[3 * NV + v] = tol * tol * bn[v];
        init[7 * NV + v] = bn[v] == 0 ? 1.0 : 0.0;
        any = any || bn[v] != 0;
    }
    if (!any) return 0;
    SVH_CUDA(cudaMemcpyAsync(pc, init.data(), init.size() * sizeof(double), cudaMemcpyHostToDevice, s));
    SVH_CUDA(cudaMemcpyAsync(r, b, nd * sizeof(double), cudaMemcpyDeviceToDevice, s));
    kcycle(S, 0, r, z, s, NVP);
    SVH_CUDA(cudaMemcpyAsync(p, z, nd * sizeof(double), cudaMemcpyDeviceToDevice, s));
    cudaGraphExec_t gx = nullptr;
    for (auto& gg : S->pcg_graphs)
        if (gg.first == NVP) gx = gg.second;
    if (!gx && s != nullptr) {
        cudaGraph_t g = nullptr;
        SVH_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        iteration();
        SVH_CUDA(cudaStreamEndCapture(s, &g));
        SVH_CUDA(cudaGraphInstantiate(&gx, g, 0));
        cudaGraphDestroy(g);
        S->pcg_graphs.push_back({NVP, gx});
    }
    constexpr int kCheck = 4;
    int it = 0;
    std::vector<double> done(NV);
    while (it < maxit) {
        const int nb = std::min(kCheck, maxit - it);
        for (int k = 0; k < nb; ++k) {
            if (gx)
                SVH_CUDA(cudaGraphLaunch(gx, s));
            else
                iteration();
        }
        it += nb;
        SVH_CUDA(cudaMemcpyAsync(done.data(), pc + 7 * NV, NV * sizeof(double), cudaMemcpyDeviceToHost, s));
        SVH_CUDA(cudaStreamSynchronize(s));
        bool all = true;
        for (int v = 0; v < NV; ++v) all = all && done[v] != 0;
        if (all) break;
    }
    return it;
}

// S^-1 of the preconditioner: AMG-preconditioned CG, or the sparse-direct comparator
static int schur_solve(svh_handle* h, const double* b, double* x, double tol, int maxit, cudaStream_t s, int NVP) {
    if (h->opts.schur_solver == 1) {
        chol_solveV(h->solve, b, x, s, NVP);
        return 1;
    }
    return pcgV(h, b, x, tol, maxit, s, NVP);
}

// out = Q^-1 in  (right preconditioner)
static void precond(svh_handle* h, const double2* in, double2* out, double tol, int maxit, cudaStream_t s) {
    Solve* S = h->solve;
    const int64_t K = h->K, n5 = 5 * K;
    double2* tt = S->d_krylov + (size_t)(2 * S->krylov_m + 3) * S->N;   // scratch vector
    SVH_LAUNCH(k_pre_e, nblk(n5), 256, 0, s, in, S->d_yinv, tt, n5);
    double* e2 = S->wbuf[4];
    double* b2 = S->wbuf[5];
    if (S->nf > 0) {
        SVH_LAUNCH(k_pre_e2, nblk(S->nf), 256, 0, s, tt, in + n5, e2, S->d_free_list, S->d_node_vox, S->d_node_axis, K,
                   S->nf);
        S->inner_its += schur_solve(h, e2, b2, tol, maxit, s, 1);
    }
    SVH_LAUNCH(k_pre_b, nblk(S->M), 256, 0, s, b2, in + n5, out + n5, S->d_node2free, S->M);
    SVH_LAUNCH(k_pre_a, nblk(K), 256, 0, s, in, out + n5, S->d_yinv, out, S->d_fnode, S->d_free, K);
}

static double cnorm(svh_handle* h, const double2* x, cudaStream_t s) {
    Solve* S = h->solve;
    SVH_LAUNCH(k_cdots, dim3(kCdotBlocks, 1), 256, 0, s, S->N, x, 0, x, reinterpret_cast<double2*>(S->d_part));
    SVH_LAUNCH(k_cdots_fin, 1, 32, 0, s, kCdotBlocks, 1, reinterpret_cast<const double2*>(S->d_part), S->d_red);
    double v[2];
    SVH_CUDA(cudaMemcpyAsync(v, S->d_red, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    SVH_CUDA(cudaStreamSynchronize(s));
    return std::sqrt(std::max(v[0], 0.0));
}

// FGMRES(m), right preconditioned; returns iterations, writes x, final true rre
static int fgmres(svh_handle* h, const double2* b, double2* x, double rre, int m, int maxit, double& final_rre,
                  cudaStream_t s) {
    Solve* S = h->solve;
    const int64_t N = S->N;
    double2* V = S->d_krylov;                         // m+1 vectors
    double2* Zp = S->d_krylov + (size_t)(m + 1) * N;  // m vectors
    double2* w = S->d_krylov + (size_t)(2 * m + 1) * N;
    double2* r = S->d_krylov + (size_t)(2 * m + 2) * N;
    double* hcol = S->d_red + 16;
    const double bnorm = cnorm(h, b, s);
    SVH_CUDA(cudaMemsetAsync(x, 0, N * sizeof(double2), s));
    if (bnorm == 0) {
        final_rre = 0;
        return 0;
    }
    int total = 0;
    final_rre = 1.0;
    const double tol_inner = h->opts.inner_tol;
    const int inner_max = h->opts.inner_maxit;
    while (total < maxit) {
        // r = b - A x
        apply_sys(h, x, w, true, s);
        SVH_LAUNCH(k_csub, nblk(N), 256, 0, s, N, b, w, r);
        const double beta = cnorm(h, r, s);
        final_rre = beta / bnorm;
        if (final_rre <= rre) break;
        SVH_LAUNCH(k_cscale, nblk(N), 256, 0, s, N, r, 1.0 / beta, V);
        std::vector<cd> H((size_t)(m + 1) * m, 0.0), cs(m), sn(m), g(m + 1, 0.0);
        g[0] = beta;
        int j = 0;
        for (; j < m && total < maxit; ++j, ++total) {
            auto c0 = std::chrono::steady_clock::now();
            precond(h, V + (size_t)j * N, Zp + (size_t)j * N, tol_inner, inner_max, s);
            SVH_CUDA(cudaStreamSynchronize(s));
            auto c1 = std::chrono::steady_clock::now();
            apply_sys(h, Zp + (size_t)j * N, w, true, s);
            SVH_CUDA(cudaStreamSynchronize(s));
            auto c2 = std::chrono::steady_clock::now();
            S->t_precond += std::chrono::duration<double>(c1 - c0).count();
            S->t_matvec += std::chrono::duration<double>(c2 - c1).count();
            // CGS2
            std::vector<cd> hj(j + 2, 0.0);
            for (int pass = 0; pass < 2; ++pass) {
                SVH_LAUNCH(k_cdots, dim3(kCdotBlocks, j + 1), 256, 0, s, N, V, N, w,
                           reinterpret_cast<double2*>(S->d_part));
                SVH_LAUNCH(k_cdots_fin, nblk(j + 1, 64), 64, 0, s, kCdotBlocks, j + 1,
                           reinterpret_cast<const double2*>(S->d_part), hcol);
                SVH_LAUNCH(k_cupdate, nblk(N), 256, 0, s, N, V, N, hcol, j + 1, w, 1.0);
                std::vector<double> hv(2 * (j + 1));
                SVH_CUDA(cudaMemcpyAsync(hv.data(), hcol, hv.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
                SVH_CUDA(cudaStreamSynchronize(s));
                for (int i = 0; i <= j; ++i) hj[i] += cd(hv[2 * i], hv[2 * i + 1]);
            }
            const double hn = cnorm(h, w, s);
            hj[j + 1] = hn;
            if (hn > 0) SVH_LAUNCH(k_cscale, nblk(N), 256, 0, s, N, w, 1.0 / hn, V + (size_t)(j + 1) * N);
            // apply previous Givens rotations
            for (int i = 0; i < j; ++i) {
                const cd t0 = std::conj(cs[i]) * hj[i] + std::conj(sn[i]) * hj[i + 1];
                const cd t1 = -sn[i] * hj[i] + cs[i] * hj[i + 1];
                hj[i] = t0;
                hj[i + 1] = t1;
            }
            const double den = std::sqrt(std::norm(hj[j]) + std::norm(hj[j + 1]));
            cs[j] = den > 0 ? hj[j] / den : cd(1.0);
            sn[j] = den > 0 ? hj[j + 1] / den : cd(0.0);
            hj[j] = den;
            hj[j + 1] = 0.0;
            g[j + 1] = -sn[j] * g[j];
            g[j] = std::conj(cs[j]) * g[j];
            for (int i = 0; i <= j; ++i) H[(size_t)i * m + j] = hj[i];
            if (std::abs(g[j + 1]) / bnorm <= rre * 0.5 || hn == 0) {
                ++j;
                ++total;
                break;
            }
        }
        // solve H y = g (upper triangular j x j)
        std::vector<cd> y(j);
        for (int i = j - 1; i >= 0; --i) {
            cd acc = g[i];
            for (int k = i + 1; k < j; ++k) acc -= H[(size_t)i * m + k] * y[k];
            y[i] = acc / H[(size_t)i * m + i];
        }
        // x += Zp y   (k_cupdate with sign -1 adds)
        std::vector<double> yv(2 * j);
        for (int i = 0; i < j; ++i) {
            yv[2 * i] = y[i].real();
            yv[2 * i + 1] = y[i].imag();
        }
        SVH_CUDA(cudaMemcpyAsync(hcol, yv.data(), yv.size() * sizeof(double), cudaMemcpyHostToDevice, s));
        SVH_LAUNCH(k_cupdate, nblk(N), 256, 0, s, N, Zp, N, hcol, j, x, -1.0);
    }
    // final true residual
    apply_sys(h, x, w, true, s);
    SVH_LAUNCH(k_csub, nblk(N), 256, 0, s, N, b, w, r);
    final_rre = cnorm(h, r, s) / bnorm;
    return total;
}

// Batched FGMRES over B ports in lockstep (time to the L-matrix): every port keeps its own
// Krylov space, Hessenberg and restart cycle, but each iteration applies the preconditioner to
// all active ports with ONE PCG on 2 NVP real right-hand sides (the AMG hierarchy, its matrices
// and the ~250-kernel cycle are shared, so the matrix traffic and launch latency are paid once
// per iteration instead of once per port) and the operator with ONE B-RHS matvec.
struct BatchWork {
    int B = 0, m = 0;
    int64_t N = 0;
    double2* kry = nullptr;   // per port: V (m+1), Z (m), w, r   -> (2m+3) N
    float2* cin = nullptr;    // [B][5K] complex64 operator input / output
    float2* cout = nullptr;
    double2* zin = nullptr;   // [B][5K] complex128 build
    double2* zout = nullptr;
    double2* base(int p) const { return kry + (size_t)p * (2 * m + 3) * N; }
    double2* V(int p, int j) const { return base(p) + (size_t)j * N; }
    double2* Z(int p, int j) const { return base(p) + (size_t)(m + 1 + j) * N; }
    double2* w(int p) const { return base(p) + (size_t)(2 * m + 1) * N; }
    double2* r(int p) const { return base(p) + (size_t)(2 * m + 2) * N; }
    void release() {
        cudaFree(kry);
        cudaFree(cin);
        cudaFree(cout);
        cudaFree(zin);
        cudaFree(zout);
        kry = nullptr;
        cin = cout = nullptr;
        zin = zout = nullptr;
    }
};

static void fgmres_batch(svh_handle* h, BatchWork& W, int nb, double2* const* bb, double2* const* xx, double rre,
                         int maxit, int NVP, std::vector<double>& final_rre, std::vector<int>& its, cudaStream_t s) {
    Solve* S = h->solve;
    const int64_t N = S->N, K = h->K, n5 = 5 * K;
    const int m = W.m;
    const double tol_inner = h->opts.inner_tol;
    const int inner_max = h->opts.inner_maxit;
    double* hcol = S->d_red + 16;
    struct St {
        double bnorm = 0;
        bool done = false;     // converged (or zero right-hand side)
        bool incycle = false;  // taking part in the current restart cycle
        int j = 0;             // Krylov vectors of the current cycle
        std::vector<cd> H, cs, sn, g;
    };
    std::vector<St> st(nb);
    final_rre.assign(nb, 1.0);
    its.assign(nb, 0);
    for (int p = 0; p < nb; ++p) {
        st[p].bnorm = cnorm(h, bb[p], s);
        SVH_CUDA(cudaMemsetAsync(xx[p], 0, N * sizeof(double2), s));
        if (st[p].bnorm == 0) {
            st[p].done = true;
            final_rre[p] = 0;
        }
    }
    double* e2 = S->wbuf[4];
    double* b2 = S->wbuf[5];
    while (true) {
        // cycle start: true residual of every unconverged port
        int nin = 0;
        for (int p = 0; p < nb; ++p) {
            St& P = st[p];
            P.incycle = false;
            if (P.done || its[p] >= maxit) continue;
            apply_sys(h, xx[p], W.w(p), true, s);
            SVH_LAUNCH(k_csub, nblk(N), 256, 0, s, N, bb[p], W.w(p), W.r(p));
            const double beta = cnorm(h, W.r(p), s);
            final_rre[p] = beta / P.bnorm;
            if (final_rre[p] <= rre) {
                P.done = true;
                continue;
            }
            SVH_LAUNCH(k_cscale, nblk(N), 256, 0, s, N, W.r(p), 1.0 / beta, W.V(p, 0));
            P.H.assign((size_t)(m + 1) * m, 0.0);
            P.cs.assign(m, 0.0);
            P.sn.assign(m, 0.0);
            P.g.assign(m + 1, 0.0);
            P.g[0] = beta;
            P.j = 0;
            P.incycle = true;
            ++nin;
        }
        if (nin == 0) break;
        for (int j = 0; j < m; ++j) {
            std::vector<int> act;
            for (int p = 0; p < nb; ++p)
                if (st[p].incycle && st[p].j == j && its[p] < maxit) act.push_back(p);
            if (act.empty()) break;
            // ---- preconditioner, all active ports at once
            SVH_CUDA(cudaMemsetAsync(e2, 0, 2 * (size_t)std::max(S->nf, 1) * NVP * sizeof(double), s));
            for (int p : act) {
                SVH_LAUNCH(k_pre_e, nblk(n5), 256, 0, s, W.V(p, j), S->d_yinv, W.w(p), n5);
                if (S->nf > 0)
                    SVH_LAUNCH(k_pre_e2V, nblk(S->nf), 256, 0, s, W.w(p), W.V(p, j) + n5, e2, S->d_free_list,
                               S->d_node_vox, S->d_node_axis, K, S->nf, NVP, p);
            }
            auto c0 = std::chrono::steady_clock::now();
            if (S->nf > 0) S->inner_its += schur_solve(h, e2, b2, tol_inner, inner_max, s, NVP);
            for (int p : act) {
                SVH_LAUNCH(k_pre_bV, nblk(S->M), 256, 0, s, b2, W.V(p, j) + n5, W.Z(p, j) + n5, S->d_node2free, S->M,
                           NVP, p);
                SVH_LAUNCH(k_pre_a, nblk(K), 256, 0, s, W.V(p, j), W.Z(p, j) + n5, S->d_yinv, W.Z(p, j), S->d_fnode,
                           S->d_free, K);
            }
            SVH_CUDA(cudaStreamSynchronize(s));
            auto c1 = std::chrono::steady_clock::now();
            // ---- operator, one matvec over the batch: w = A Z_j
            if (h->opts.precision == 1) {   // complex128 build: fp64 operator on the stacked Z_j
                for (int p : act)
                    SVH_CUDA(cudaMemcpyAsync(W.zin + (size_t)p * n5, W.Z(p, j), n5 * sizeof(double2),
                                             cudaMemcpyDeviceToDevice, s));
                matvec_z(h, W.zin, W.zout, nb, false, s);
            } else {
                for (int p : act) SVH_LAUNCH(k_to_c64, nblk(n5), 256, 0, s, W.Z(p, j), W.cin + (size_t)p * n5, n5);
                matvec(h, W.cin, W.cout, nb, false, true, s);
            }
            for (int p : act) {
                if (h->opts.precision == 1)
                    SVH_LAUNCH(k_sys_I<double2>, nblk(K), 256, 0, s, W.zout + (size_t)p * n5, W.Z(p, j), W.w(p),
                               S->d_fnode, S->d_free, K);
                else
                    SVH_LAUNCH(k_sys_I<float2>, nblk(K), 256, 0, s, W.cout + (size_t)p * n5, W.Z(p, j), W.w(p),
                               S->d_fnode, S->d_free, K);
                SVH_LAUNCH(k_sys_Phi, nblk(S->M), 256, 0, s, W.Z(p, j), W.w(p), S->d_node_vox, S->d_node_axis,
                           S->d_free, K, S->M);
            }
            SVH_CUDA(cudaStreamSynchronize(s));
            auto c2 = std::chrono::steady_clock::now();
            S->t_precond += std::chrono::duration<double>(c1 - c0).count();
            S->t_matvec += std::chrono::duration<double>(c2 - c1).count();
            // ---- per port: CGS2 and the Givens update (host)
            for (int p : act) {
                St& P = st[p];
                double2* V = W.V(p, 0);
                double2* w = W.w(p);
                std::vector<cd> hj(j + 2, 0.0);
                for (int pass = 0; pass < 2; ++pass) {
                    SVH_LAUNCH(k_cdots, dim3(kCdotBlocks, j + 1), 256, 0, s, N, V, N, w,
                               reinterpret_cast<double2*>(S->d_part));
                    SVH_LAUNCH(k_cdots_fin, nblk(j + 1, 64), 64, 0, s, kCdotBlocks, j + 1,
                               reinterpret_cast<const double2*>(S->d_part), hcol);
                    SVH_LAUNCH(k_cupdate, nblk(N), 256, 0, s, N, V, N, hcol, j + 1, w, 1.0);
                    std::vector<double> hv(2 * (j + 1));
                    SVH_CUDA(cudaMemcpyAsync(hv.data(), hcol, hv.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
                    SVH_CUDA(cudaStreamSynchronize(s));
                    for (int i = 0; i <= j; ++i) hj[i] += cd(hv[2 * i], hv[2 * i + 1]);
                }
                const double hn = cnorm(h, w, s);
                hj[j + 1] = hn;
                if (hn > 0) SVH_LAUNCH(k_cscale, nblk(N), 256, 0, s, N, w, 1.0 / hn, W.V(p, j + 1));
                for (int i = 0; i < j; ++i) {
                    const cd t0 = std::conj(P.cs[i]) * hj[i] + std::conj(P.sn[i]) * hj[i + 1];
                    const cd t1 = -P.sn[i] * hj[i] + P.cs[i] * hj[i + 1];
                    hj[i] = t0;
                    hj[i + 1] = t1;
                }
                const double den = std::sqrt(std::norm(hj[j]) + std::norm(hj[j + 1]));
                P.cs[j] = den > 0 ? hj[j] / den : cd(1.0);
                P.sn[j] = den > 0 ? hj[j + 1] / den : cd(0.0);
                hj[j] = den;
                hj[j + 1] = 0.0;
                P.g[j + 1] = -P.sn[j] * P.g[j];
                P.g[j] = std::conj(P.cs[j]) * P.g[j];
                for (int i = 0; i <= j; ++i) P.H[(size_t)i * m + j] = hj[i];
                P.j = j + 1;
                ++its[p];
                if (std::abs(P.g[j + 1]) / P.bnorm <= rre * 0.5 || hn == 0) P.incycle = false;   // cycle ends
            }
        }
        // ---- cycle end: x_p += Z_p y_p
        for (int p = 0; p < nb; ++p) {
            St& P = st[p];
            if (P.done || P.j == 0) continue;
            const int jj = P.j;
            std::vector<cd> y(jj);
            for (int i = jj - 1; i >= 0; --i) {
                cd acc = P.g[i];
                for (int k = i + 1; k < jj; ++k) acc -= P.H[(size_t)i * m + k] * y[k];
                y[i] = acc / P.H[(size_t)i * m + i];
            }
            std::vector<double> yv(2 * jj);
            for (int i = 0; i < jj; ++i) {
                yv[2 * i] = y[i].real();
                yv[2 * i + 1] = y[i].imag();
            }
            SVH_CUDA(cudaMemcpyAsync(hcol, yv.data(), yv.size() * sizeof(double), cudaMemcpyHostToDevice, s));
            SVH_LAUNCH(k_cupdate, nblk(N), 256, 0, s, N, W.Z(p, 0), N, hcol, jj, xx[p], -1.0);
            SVH_CUDA(cudaStreamSynchronize(s));
            P.j = 0;
        }
    }
    // final true residuals
    for (int p = 0; p < nb; ++p) {
        if (st[p].bnorm == 0) continue;
        apply_sys(h, xx[p], W.w(p), true, s);
        SVH_LAUNCH(k_csub, nblk(N), 256, 0, s, N, bb[p], W.w(p), W.r(p));
        final_rre[p] = cnorm(h, W.r(p), s) / st[p].bnorm;
    }
}

// ---------------------------------------------------------------------------
struct PortSets {
    std::vector<std::vector<int32_t>> plus, minus;
    std::vector<int32_t> fixed;
};

static std::vector<int32_t> rect_nodes(svh_handle* h, const svh_face_rect* rects, int n) {
    Solve* S = h->solve;
    std::vector<int32_t> out;
    for (int i = 0; i < n; ++i) {
        const svh_face_rect& R = rects[i];
        SVH_CHECK(R.axis >= 0 && R.axis < 3 && (R.side == 1 || R.side == -1), SVH_EINVAL, "bad face rect");
        for (int z = std::max(0, R.lo[2]); z < std::min(h->kz, R.hi[2]); ++z)
            for (int y = std::max(0, R.lo[1]); y < std::min(h->ky, R.hi[1]); ++y)
                for (int x = std::max(0, R.lo[0]); x < std::min(h->kx, R.hi[0]); ++x) {
                    const int32_t k = h->h_vmap[((int64_t)z * h->ky + y) * h->kx + x];
                    if (k < 0) continue;
                    out.push_back(S->fnode[6 * k + 2 * R.axis + (R.side > 0)]);
                }
    }
    std::sort(out.begin(), out.end());
    out.erase(std::unique(out.begin(), out.end()), out.end());
    return out;
}

static PortSets port_sets(svh_handle* h, const svh_port* ports, int P) {
    Solve* S = h->solve;
    PortSets ps;
    for (int p = 0; p < P; ++p) {
        ps.plus.push_back(rect_nodes(h, ports[p].plus, ports[p].n_plus));
        ps.minus.push_back(rect_nodes(h, ports[p].minus, ports[p].n_minus));
        SVH_CHECK(!ps.plus.back().empty() && !ps.minus.back().empty(), SVH_EINVAL,
                  "port " + std::to_string(p) + " has an empty terminal");
        ps.fixed.insert(ps.fixed.end(), ps.plus.back().begin(), ps.plus.back().end());
        ps.fixed.insert(ps.fixed.end(), ps.minus.back().begin(), ps.minus.back().end());
    }
    std::sort(ps.fixed.begin(), ps.fixed.end());
    ps.fixed.erase(std::unique(ps.fixed.begin(), ps.fixed.end()), ps.fixed.end());
    // G14: ground one node of every voxel component without a fixed node (union-find over shared faces)
    std::vector<int32_t> parent(h->K);
    std::iota(parent.begin(), parent.end(), 0);
    std::function<int32_t(int32_t)> find = [&](int32_t a) {
        while (parent[a] != a) a = parent[a] = parent[parent[a]];
        return a;
    };
    for (int64_t r = 0; r < S->M; ++r) {
        const int32_t v = S->node_vox[2 * r], u = S->node_vox[2 * r + 1];
        if (v >= 0 && u >= 0) parent[find(v)] = find(u);
    }
    std::vector<uint8_t> has_fixed(h->K, 0);
    for (int32_t r : ps.fixed) {
        const int32_t v = S->node_vox[2 * r] >= 0 ? S->node_vox[2 * r] : S->node_vox[2 * r + 1];
        has_fixed[find(v)] = 1;
    }
    std::vector<int32_t> extra;
    for (int64_t k = 0; k < h->K; ++k) {
        const int32_t root = find((int32_t)k);
        if (!has_fixed[root]) {
            has_fixed[root] = 1;
            extra.push_back(S->fnode[6 * k + 0]);
        }
    }
    ps.fixed.insert(ps.fixed.end(), extra.begin(), extra.end());
    std::sort(ps.fixed.begin(), ps.fixed.end());
    ps.fixed.erase(std::unique(ps.fixed.begin(), ps.fixed.end()), ps.fixed.end());
    return ps;
}

static void ensure_structure(svh_handle* h) {
    if (!h->solve) build_structure(h);
}

static void solve_columns(svh_handle* h, const svh_port* ports, int P, const int32_t* sel, int nsel, double* Ycols,
                          svh_stats* st) {
    ensure_structure(h);
    Solve* S = h->solve;
    auto t0 = std::chrono::steady_clock::now();
    PortSets ps = port_sets(h, ports, P);
    const int m = std::max(1, h->opts.restart);
    // batched multi-port solve (lockstep FGMRES, one shared PCG): batch size by memory, <= 16
    int Bmax = std::min(nsel, 16);
    if (Bmax > 1) {
        ensure_structure(h);
        size_t fr = 0, tt = 0;
        cudaMemGetInfo(&fr, &tt);
        const size_t per = (size_t)(2 * m + 5) * S->N * sizeof(double2) + (size_t)10 * h->K * sizeof(float2);
        Bmax = std::max(1, std::min(Bmax, (int)(0.5 * (double)fr / (double)per)));
    }
    int NVP = 1;
    while (NVP < Bmax) NVP <<= 1;
    build_amg(h, ps.fixed, NVP);
    ensure_work(h, m);
    if (!S->stream) SVH_CUDA(cudaStreamCreateWithFlags(&S->stream, cudaStreamNonBlocking));
    if (!S->d_pcg || S->pcg_cap < S->nvp_cap) {
        drop_pcg_graph(S);
        cudaFree(S->d_pcg);
        SVH_CUDA(cudaMalloc(&S->d_pcg, 16 * (size_t)S->nvp_cap * sizeof(double)));
        S->pcg_cap = S->nvp_cap;
    }
    cudaStream_t s = S->stream;
    SVH_CUDA(cudaDeviceSynchronize());   // setup copies (legacy stream) before the non-blocking stream
    const int64_t N = S->N;
    double2* b = S->d_krylov + (size_t)(2 * m + 3) * N;   // scratch slot (also used by precond -> copy out first)
    double2* x = nullptr;
    SVH_CUDA(cudaMalloc(&x, N * sizeof(double2)));
    double2* bb = nullptr;
    SVH_CUDA(cudaMalloc(&bb, N * sizeof(double2)));
    uint8_t* pm = nullptr;
    SVH_CUDA(cudaMalloc(&pm, S->M));
    int32_t* dnodes = nullptr;
    size_t maxn = 1;
    for (int p = 0; p < P; ++p) maxn = std::max(maxn, ps.plus[p].size());
    SVH_CUDA(cudaMalloc(&dnodes, maxn * sizeof(int32_t)));
    double* cur = nullptr;
    SVH_CUDA(cudaMalloc(&cur, 2 * sizeof(double)));
    bool all_conv = true;
    double worst = 0;
    int tot_it = 0;
    S->inner_its = 0;
    S->t_matvec = S->t_precond = 0;
    (void)b;
    auto port_currents = [&](const double2* xs, int si) {
        for (int q = 0; q < P; ++q) {
            SVH_CUDA(cudaMemcpyAsync(dnodes, ps.plus[q].data(), ps.plus[q].size() * sizeof(int32_t),
                                     cudaMemcpyHostToDevice, s));
            SVH_LAUNCH(k_port_current, 1, 256, 0, s, xs, dnodes, (int)ps.plus[q].size(), S->d_node_vox,
                       S->d_node_axis, h->K, cur);
            double c2[2];
            SVH_CUDA(cudaMemcpyAsync(c2, cur, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
            SVH_CUDA(cudaStreamSynchronize(s));
            Ycols[2 * ((size_t)si * P + q)] = c2[0];
            Ycols[2 * ((size_t)si * P + q) + 1] = c2[1];
        }
    };
    if (Bmax > 1) {
        BatchWork W;
        W.B = Bmax;
        W.m = m;
        W.N = N;
        std::vector<double2*> bbs(Bmax, nullptr), xs(Bmax, nullptr);
        auto release = [&] {
            W.release();
            for (auto q : bbs) cudaFree(q);
            for (auto q : xs) cudaFree(q);
        };
        try {
            SVH_CUDA(cudaMalloc(&W.kry, (size_t)Bmax * (2 * m + 3) * N * sizeof(double2)));
            SVH_CUDA(cudaMalloc(&W.cin, (size_t)Bmax * 5 * h->K * sizeof(float2)));
            SVH_CUDA(cudaMalloc(&W.cout, (size_t)Bmax * 5 * h->K * sizeof(float2)));
            SVH_CUDA(cudaMemsetAsync(W.cin, 0, (size_t)Bmax * 5 * h->K * sizeof(float2), s));
            if (h->opts.precision == 1) {
                SVH_CUDA(cudaMalloc(&W.zin, (size_t)Bmax * 5 * h->K * sizeof(double2)));
                SVH_CUDA(cudaMalloc(&W.zout, (size_t)Bmax * 5 * h->K * sizeof(double2)));
                SVH_CUDA(cudaMemsetAsync(W.zin, 0, (size_t)Bmax * 5 * h->K * sizeof(double2), s));
            }
            for (int p = 0; p < Bmax; ++p) {
                SVH_CUDA(cudaMalloc(&bbs[p], N * sizeof(double2)));
                SVH_CUDA(cudaMalloc(&xs[p], N * sizeof(double2)));
            }
            for (int s0 = 0; s0 < nsel; s0 += Bmax) {
                const int nb = std::min(Bmax, nsel - s0);
                for (int k = 0; k < nb; ++k) {
                    const int p = sel[s0 + k];
                    SVH_CHECK(p >= 0 && p < P, SVH_EINVAL, "bad port index");
                    std::vector<uint8_t> mask(S->M, 0);
                    for (int32_t r : ps.plus[p]) mask[r] = 1;
                    SVH_CUDA(cudaMemcpyAsync(pm, mask.data(), S->M, cudaMemcpyHostToDevice, s));
                    SVH_LAUNCH(k_rhs, nblk(h->K + S->M), 256, 0, s, bbs[k], pm, S->d_fnode, h->K, S->M);
                    SVH_CUDA(cudaStreamSynchronize(s));   // pm is reused by the next port
                }
                std::vector<double> rres;
                std::vector<int> itv;
                fgmres_batch(h, W, nb, bbs.data(), xs.data(), h->opts.rre, h->opts.max_iters, NVP, rres, itv, s);
                for (int k = 0; k < nb; ++k) {
                    tot_it += itv[k];
                    worst = std::max(worst, rres[k]);
                    if (!(rres[k] <= h->opts.rre * 1.0001)) all_conv = false;
                    if (st) st->iterations = itv[k];
                    port_currents(xs[k], s0 + k);
                }
            }
        } catch (...) {
            release();
            cudaFree(x);
            cudaFree(bb);
            cudaFree(pm);
            cudaFree(dnodes);
            cudaFree(cur);
            throw;
        }
        release();
        nsel = 0;   // done
    }
    for (int si = 0; si < nsel; ++si) {
        const int p = sel[si];
        SVH_CHECK(p >= 0 && p < P, SVH_EINVAL, "bad port index");
        std::vector<uint8_t> mask(S->M, 0);
        for (int32_t r : ps.plus[p]) mask[r] = 1;
        // stream-ordered H2D (a pageable cudaMemcpy may return before its DMA lands, and
        // the solve stream does not wait for the legacy stream)
        SVH_CUDA(cudaMemcpyAsync(pm, mask.data(), S->M, cudaMemcpyHostToDevice, s));
        SVH_LAUNCH(k_rhs, nblk(h->K + S->M), 256, 0, s, bb, pm, S->d_fnode, h->K, S->M);
        double rre_out = 0;
        const int its = fgmres(h, bb, x, h->opts.rre, m, h->opts.max_iters, rre_out, s);
        tot_it += its;
        worst = std::max(worst, rre_out);
        if (!(rre_out <= h->opts.rre * 1.0001)) all_conv = false;
        if (st) st->iterations = its;
        port_currents(x, si);
    }
    SVH_CUDA(cudaStreamSynchronize(s));
    cudaFree(x);
    cudaFree(bb);
    cudaFree(pm);
    cudaFree(dnodes);
    cudaFree(cur);
    if (st) {
        st->total_iterations += tot_it;
        st->inner_iterations += S->inner_its;
        st->t_matvec_s += S->t_matvec;
        st->t_precond_s += S->t_precond;
        st->t_precond_setup_s = S->t_pre_setup;
        st->precond_bytes = S->pre_bytes;
        st->schur_solver = h->opts.schur_solver;
        st->amg_levels = h->opts.schur_solver == 1 ? 0 : (int32_t)S->levels.size();
        st->amg_op_complexity = h->opts.schur_solver == 1 ? 0.0 : S->op_complexity;
        st->converged = all_conv ? 1 : 0;
        st->final_rre = std::max(st->final_rre, worst);
        st->t_solve_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        st->t_setup_s = h->t_setup;
    }
    if (!all_conv) throw Error{SVH_ENOCONV, "GMRES did not reach rre (best iterate returned)"};
}

}  // namespace svh

using namespace svh;
extern "C" {

int svh_apply_system(svh_handle* h, const void* x, void* y, int32_t nrhs, svh_stream stream) {
    try {
        SVH_CHECK(h && x && y && nrhs >= 1 && x != y, SVH_EINVAL, "bad args");
        SVH_CUDA(cudaSetDevice(h->device));
        ensure_structure(h);
        Solve* S = h->solve;
        cudaStream_t s = (cudaStream_t)stream;
        const int64_t N = S->N, K = h->K;
        float2* zi = nullptr;
        SVH_CUDA(cudaMalloc(&zi, 5 * K * nrhs * sizeof(float2)));
        float2* xin = nullptr;
        SVH_CUDA(cudaMalloc(&xin, 5 * K * nrhs * sizeof(float2)));
        for (int r = 0; r < nrhs; ++r)
            SVH_CUDA(cudaMemcpyAsync(xin + 5 * K * r, (const float2*)x + N * r, 5 * K * sizeof(float2),
                                     cudaMemcpyDeviceToDevice, s));
        matvec(h, xin, zi, nrhs, false, true, s);
        for (int r = 0; r < nrhs; ++r)
            SVH_LAUNCH(k_sys_c64, nblk(K + S->M), 256, 0, s, zi + 5 * K * r, (const float2*)x + N * r,
                       (float2*)y + N * r, S->d_fnode, S->d_node_vox, S->d_node_axis, K, S->M);
        SVH_CUDA(cudaStreamSynchronize(s));
        cudaFree(zi);
        cudaFree(xin);
        return SVH_OK;
    }
    SVH_C_ABI_CATCH
}

int svh_solve_columns(svh_handle* h, const svh_port* ports, int32_t n_ports, const int32_t* sel, int32_t n_sel,
                      double* Y_cols, svh_stats* stats) {
    try {
        SVH_CHECK(h && ports && n_ports >= 1 && sel && n_sel >= 0 && Y_cols, SVH_EINVAL, "bad args");
        SVH_CUDA(cudaSetDevice(h->device));
        if (stats) std::memset(stats, 0, sizeof(*stats));
        solve_columns(h, ports, n_ports, sel, n_sel, Y_cols, stats);
        return SVH_OK;
    }
    SVH_C_ABI_CATCH
}

int svh_solve(svh_handle* h, const svh_port* ports, int32_t n_ports, double* Z_port, double* L_H, double* R_ohm,
              double* Y_port, svh_stats* stats) {
    int code = SVH_OK;
    try {
        SVH_CHECK(h && ports && n_ports >= 1, SVH_EINVAL, "bad args");
        SVH_CUDA(cudaSetDevice(h->device));
        if (stats) std::memset(stats, 0, sizeof(*stats));
        const int P = n_ports;
        std::vector<int32_t> sel(P);
        std::iota(sel.begin(), sel.end(), 0);
        std::vector<double> Yc((size_t)2 * P * P);
        try {
            solve_columns(h, ports, P, sel.data(), P, Yc.data(), stats);
        } catch (const Error& e) {
            if (e.code != SVH_ENOCONV) throw;
            code = SVH_ENOCONV;
            set_error(e.msg);
        }
        // Y[q][p] = column p entry q
        std::vector<double> Yr((size_t)2 * P * P);
        for (int p = 0; p < P; ++p)
            for (int q = 0; q < P; ++q) {
                Yr[2 * ((size_t)q * P + p)] = Yc[2 * ((size_t)p * P + q)];
                Yr[2 * ((size_t)q * P + p) + 1] = Yc[2 * ((size_t)p * P + q) + 1];
            }
        if (Y_port) std::memcpy(Y_port, Yr.data(), Yr.size() * sizeof(double));
        const int c2 = svh_y_to_zl(Yr.data(), P, h->freq, Z_port, L_H, R_ohm);
        if (c2 != SVH_OK) return c2;
        return code;
    }
    SVH_C_ABI_CATCH
}

int svh_y_to_zl(const double* Yp, int32_t P, double freq_hz, double* Z_port, double* L_H, double* R_ohm) {
    try {
        SVH_CHECK(Yp && P >= 1 && freq_hz > 0, SVH_EINVAL, "bad args");
        const double omega = 2.0 * M_PI * freq_hz;
        // Z = Y^-1 (Gauss-Jordan with partial pivoting)
        std::vector<cd> Aug((size_t)P * 2 * P);
        for (int i = 0; i < P; ++i)
            for (int j = 0; j < P; ++j) {
                Aug[(size_t)i * 2 * P + j] = cd(Yp[2 * ((size_t)i * P + j)], Yp[2 * ((size_t)i * P + j) + 1]);
                Aug[(size_t)i * 2 * P + P + j] = (i == j) ? 1.0 : 0.0;
            }
        for (int c = 0; c < P; ++c) {
            int piv = c;
            for (int i = c + 1; i < P; ++i)
                if (std::abs(Aug[(size_t)i * 2 * P + c]) > std::abs(Aug[(size_t)piv * 2 * P + c])) piv = i;
            SVH_CHECK(std::abs(Aug[(size_t)piv * 2 * P + c]) > 1e-300, SVH_EOPENPORT, "singular Y (open port)");
            if (piv != c)
                for (int j = 0; j < 2 * P; ++j) std::swap(Aug[(size_t)c * 2 * P + j], Aug[(size_t)piv * 2 * P + j]);
            const cd d = Aug[(size_t)c * 2 * P + c];
            for (int j = 0; j < 2 * P; ++j) Aug[(size_t)c * 2 * P + j] /= d;
            for (int i = 0; i < P; ++i) {
                if (i == c) continue;
                const cd f = Aug[(size_t)i * 2 * P + c];
                if (f == 0.0) continue;
                for (int j = 0; j < 2 * P; ++j) Aug[(size_t)i * 2 * P + j] -= f * Aug[(size_t)c * 2 * P + j];
            }
        }
        for (int i = 0; i < P; ++i)
            for (int j = 0; j < P; ++j) {
                const cd z = Aug[(size_t)i * 2 * P + P + j];
                const size_t k = (size_t)i * P + j;
                if (Z_port) {
                    Z_port[2 * k] = z.real();
                    Z_port[2 * k + 1] = z.imag();
                }
                if (L_H) L_H[k] = z.imag() / omega;
                if (R_ohm) R_ohm[k] = z.real();
            }
        return SVH_OK;
    }
    SVH_C_ABI_CATCH
}

}  // extern "C"
