// H2: the 7 unit-voxel Galerkin kernels, fp64 quadrature on the GPU.
//
// Z_green^{b,a}_{lk} = j w mu0 dx T^{b,a}(l - k) (dx^5 law App. B
// P:343 with the G1 basis normalisation).  Every block T^{b,a} is a signed
// combination of 7 reduced kernels:
//   K(m; Wx, Wy, Wz) = 1/(4 pi) int_{[-1,1]^3} Wx(sx) Wy(sy) Wz(sz) / |s + m| ds
//   W0(s) = 1 - |s|,  W1(s) = -s (1 - |s|)/2,  W2(s) = 1/12 - |s|/4 + |s|^3/6
//   K0 = K(W0,W0,W0), K1c = W1 on axis c, K2c = W2 on axis c.
// Only non-negative offsets are computed (K0, K2c even; K1c odd on axis c).
//
// Quadrature: the 8 unit sub-cubes of [-1,1]^3 (the |s| kinks lie on their
// faces).  Offsets with max|m| <= 1 ("near", at most 8 of them): sub-cubes
// having the singular point -m as a vertex use a Duffy map (3 pyramids,
// Jacobian u^2 cancels 1/r), GL order 20; the others GL 20.  Far offsets:
// one thread per offset, tensor GL per sub-cube with order by distance.
#include <cmath>
#include <vector>

#include "internal.h"

namespace svh {

namespace {
constexpr int kMaxN = 24;
struct GL {
    double x[kMaxN + 1][kMaxN];   // nodes on [0,1]
    double w[kMaxN + 1][kMaxN];
};

void legendre_rule(int n, double* x01, double* w01) {
    // Newton on P_n with the three-term recurrence; nodes mapped to [0,1]
    for (int i = 0; i < n; ++i) {
        double z = std::cos(M_PI * (i + 0.75) / (n + 0.5));
        double pp = 0;
        for (int it = 0; it < 100; ++it) {
            double p1 = 1, p2 = 0;
            for (int j = 1; j <= n; ++j) {
                double p3 = p2;
                p2 = p1;
                p1 = ((2.0 * j - 1) * z * p2 - (j - 1.0) * p3) / j;
            }
            pp = n * (z * p1 - p2) / (z * z - 1.0);
            double z1 = z;
            z = z1 - p1 / pp;
            if (std::fabs(z - z1) < 1e-16) break;
        }
        x01[i] = 0.5 * (1.0 - z);
        w01[i] = 1.0 / ((1.0 - z * z) * pp * pp);   // = 0.5 * 2/((1-z^2) P'^2)
    }
}

__device__ __forceinline__ void wfun(double s, double& w0, double& w1, double& w2) {
    const double a = fabs(s);
    w0 = 1.0 - a;
    w1 = -s * (1.0 - a) * 0.5;
    w2 = 1.0 / 12.0 - a * 0.25 + a * a * a * (1.0 / 6.0);
}

__device__ __forceinline__ int far_order(int mx, int my, int mz) {
    const double dx = fmax(mx - 1.0, 0.0), dy = fmax(my - 1.0, 0.0), dz = fmax(mz - 1.0, 0.0);
    const double d = sqrt(dx * dx + dy * dy + dz * dz);
    return d < 1.5 ? 12 : d < 3.0 ? 10 : d < 6.0 ? 8 : d < 12.0 ? 6 : d < 40.0 ? 5 : 4;
}

// far offsets: one thread per offset
__global__ void k_quad_far(double* __restrict__ out, int Kx, int Ky, int Kz, const GL* __restrict__ gl) {
    const int64_t Kt = (int64_t)Kx * Ky * Kz;
    const int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (id >= Kt) return;
    const int mx = (int)(id % Kx), my = (int)((id / Kx) % Ky), mz = (int)(id / ((int64_t)Kx * Ky));
    if (mx <= 1 && my <= 1 && mz <= 1) return;
    const int n = far_order(mx, my, mz);
    const double* xs = gl->x[n];
    const double* ws = gl->w[n];
    double acc[7] = {0, 0, 0, 0, 0, 0, 0};
    for (int cz = -1; cz <= 0; ++cz)
        for (int cy = -1; cy <= 0; ++cy)
            for (int cx = -1; cx <= 0; ++cx) {
                for (int k = 0; k < n; ++k) {
                    const double sz = cz + xs[k];
                    double z0, z1, z2;
                    wfun(sz, z0, z1, z2);
                    const double dz = sz + mz;
                    for (int j = 0; j < n; ++j) {
                        const double sy = cy + xs[j];
                        double y0, y1, y2;
                        wfun(sy, y0, y1, y2);
                        const double dy = sy + my;
                        const double wjk = ws[j] * ws[k];
                        for (int i = 0; i < n; ++i) {
                            const double sx = cx + xs[i];
                            double x0, x1, x2;
                            wfun(sx, x0, x1, x2);
                            const double ddx = sx + mx;
                            const double f = ws[i] * wjk * rsqrt(ddx * ddx + dy * dy + dz * dz);
                            const double fyz = f * y0 * z0;
                            acc[0] += fyz * x0;
                            acc[1] += fyz * x1;
                            acc[4] += fyz * x2;
                            const double fx = f * x0;
                            acc[2] += fx * y1 * z0;
                            acc[5] += fx * y2 * z0;
                            acc[3] += fx * y0 * z1;
                            acc[6] += fx * y0 * z2;
                        }
                    }
                }
            }
    const double s = 1.0 / (4.0 * M_PI);
    for (int q = 0; q < 7; ++q) out[q * Kt + id] = acc[q] * s;
}

// near offsets (max |m| <= 1): one CTA per offset, Duffy on vertex sub-cubes
__global__ void k_quad_near(double* __restrict__ out, int Kx, int Ky, int Kz, const GL* __restrict__ gl, int n) {
    const int64_t Kt = (int64_t)Kx * Ky * Kz;
    const int mx = blockIdx.x & 1, my = (blockIdx.x >> 1) & 1, mz = (blockIdx.x >> 2) & 1;
    if (mx >= Kx || my >= Ky || mz >= Kz) return;
    const int64_t id = ((int64_t)mz * Ky + my) * Kx + mx;
    const double* xs = gl->x[n];
    const double* ws = gl->w[n];
    const double m[3] = {(double)mx, (double)my, (double)mz};
    const double p[3] = {-m[0], -m[1], -m[2]};
    double acc[7] = {0, 0, 0, 0, 0, 0, 0};
    const int n3 = n * n * n;
    for (int sc = 0; sc < 8; ++sc) {
        const double lo[3] = {(sc & 1) ? 0.0 : -1.0, (sc & 2) ? 0.0 : -1.0, (sc & 4) ? 0.0 : -1.0};
        bool vertex = true;
        double sgn[3];
        for (int a = 0; a < 3; ++a) {
            if (p[a] == lo[a]) sgn[a] = 1.0;
            else if (p[a] == lo[a] + 1.0) sgn[a] = -1.0;
            else vertex = false;
        }
        const int npts = vertex ? 3 * n3 : n3;
        for (int t = threadIdx.x; t < npts; t += blockDim.x) {
            double s[3], w;
            const int pyr = t / n3, r = t - pyr * n3;
            const int i = r % n, j = (r / n) % n, k = r / (n * n);
            if (vertex) {
                const double u = xs[i], v = xs[j], ww = xs[k];
                double tt[3];
                const int a0 = pyr, a1 = (pyr + 1) % 3, a2 = (pyr + 2) % 3;
                tt[a0] = u;
                tt[a1] = u * v;
                tt[a2] = u * ww;
                for (int a = 0; a < 3; ++a) s[a] = p[a] + sgn[a] * tt[a];
                w = ws[i] * ws[j] * ws[k] * u * u;
            } else {
                s[0] = lo[0] + xs[i];
                s[1] = lo[1] + xs[j];
                s[2] = lo[2] + xs[k];
                w = ws[i] * ws[j] * ws[k];
            }
            const double d0 = s[0] + m[0], d1 = s[1] + m[1], d2 = s[2] + m[2];
            const double f = w / sqrt(d0 * d0 + d1 * d1 + d2 * d2);
            double x0, x1, x2, y0, y1, y2, z0, z1, z2;
            wfun(s[0], x0, x1, x2);
            wfun(s[1], y0, y1, y2);
            wfun(s[2], z0, z1, z2);
            acc[0] += f * x0 * y0 * z0;
            acc[1] += f * x1 * y0 * z0;
            acc[2] += f * x0 * y1 * z0;
            acc[3] += f * x0 * y0 * z1;
            acc[4] += f * x2 * y0 * z0;
            acc[5] += f * x0 * y2 * z0;
            acc[6] += f * x0 * y0 * z2;
        }
    }
    __shared__ double red[7][256];
    for (int q = 0; q < 7; ++q) red[q][threadIdx.x] = acc[q];
    __syncthreads();
    for (int st = blockDim.x / 2; st > 0; st >>= 1) {
        if (threadIdx.x < st)
            for (int q = 0; q < 7; ++q) red[q][threadIdx.x] += red[q][threadIdx.x + st];
        __syncthreads();
    }
    if (threadIdx.x == 0)
        for (int q = 0; q < 7; ++q) out[q * Kt + id] = red[q][0] / (4.0 * M_PI);
}
}  // namespace

void compute_kernels(svh_handle* h) {
    GL host{};
    for (int n = 1; n <= kMaxN; ++n) legendre_rule(n, host.x[n], host.w[n]);
    GL* dgl = nullptr;
    SVH_CUDA(cudaMalloc(&dgl, sizeof(GL)));
    SVH_CUDA(cudaMemcpy(dgl, &host, sizeof(GL), cudaMemcpyHostToDevice));
    SVH_CUDA(cudaMalloc(&h->d_kern, sizeof(double) * 7 * h->Kt));
    const int bs = 128;
    const int64_t nb = (h->Kt + bs - 1) / bs;
    SVH_LAUNCH(k_quad_far, dim3((unsigned)nb), bs, 0, 0, h->d_kern, h->kx, h->ky, h->kz, dgl);
    SVH_LAUNCH(k_quad_near, dim3(8), 256, 0, 0, h->d_kern, h->kx, h->ky, h->kz, dgl, 20);
    SVH_CUDA(cudaDeviceSynchronize());
    cudaFree(dgl);
}

}  // namespace svh
