"""Oracle: port excitation, dense saddle solve (Eq. 7) and inductance extraction.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The method solves Eq. 7 iteratively (GMRES(50)) with the Schur
preconditioner of Eq. 12-15; the iteration converges to the exact solution of
the linear system, so the oracle is a direct dense solve (numpy LU).

Readings (the paper defers V, Phi and ports to [18]):
* G12 sign: with A = outward-flux incidence (oracle/lattice.py), Galerkin
  testing of -grad(Phi) gives Z I + A^T Phi = 0 on every basis row; continuity
  (Eq. 2) gives A I = 0 on every free node.  This is Eq. 7 with Phi -> -Phi.
* G13 ports: Dirichlet potentials on port face nodes -- 1 V on the + faces of
  the driven port, 0 V on its - faces and on every face of the other ports
  (common ground); KCL rows only at free nodes.  Port current = current
  entering the conductor through the + faces = -sum_{r in +faces} (A I)_r.
  Y[:, p] = port currents for a 1 V drive of port p; Z = Y^-1; L = Im Z / w;
  R = Re Z.
* G14: a connected conductor touching no port face gets one node grounded.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
from scipy.sparse.csgraph import connected_components

from .lattice import Lattice
from .operator import dense_Z


def port_nodes(lat: Lattice, rects):
    """Node ids of a face set [(axis, side, lo, hi), ...] (faces of empty voxels ignored)."""
    out = []
    for axis, side, lo, hi in rects:
        xs, ys, zs = [np.arange(lo[d], hi[d]) for d in range(3)]
        X, Y, Z = np.meshgrid(xs, ys, zs, indexing="ij")
        cells = np.stack([X.ravel(), Y.ravel(), Z.ravel()], 1)
        occ = lat.occ[cells[:, 2], cells[:, 1], cells[:, 0]]
        cells = cells[occ]
        if cells.size:
            out.append(lat.face_node(axis, cells, side))
    return np.unique(np.concatenate(out)) if out else np.zeros(0, dtype=np.int64)


def floating_ground_nodes(lat: Lattice, fixed):
    """G14: one node of every voxel-connected component that has no fixed node."""
    A = lat.incidence()
    # voxel adjacency through shared faces: node-voxel incidence
    rows, cols = (A != 0).nonzero()
    vox = cols % lat.K
    NV = sp.coo_matrix((np.ones(rows.size), (rows, vox)), shape=(lat.M, lat.K)).tocsr()
    adj = (NV.T @ NV)
    ncomp, lab = connected_components(adj, directed=False)
    fixed_vox = set(lab[np.unique(vox[np.isin(rows, fixed)])]) if len(fixed) else set()
    extra = []
    for c in range(ncomp):
        if c in fixed_vox:
            continue
        k = int(np.nonzero(lab == c)[0][0])
        extra.append(int(lat.face_node(0, lat.coords[k], -1)))
    return np.array(extra, dtype=np.int64)


def solve_ports(lat: Lattice, materials, omega: float, dx: float, ports, return_fields=False):
    """Dense direct solve of the reduced saddle system for every port (G13)."""
    A = lat.incidence().toarray()
    Z = dense_Z(lat, materials, omega, dx)
    plus = [port_nodes(lat, p["plus"]) for p in ports]
    minus = [port_nodes(lat, p["minus"]) for p in ports]
    for q in range(len(ports)):
        if plus[q].size == 0 or minus[q].size == 0:
            raise ValueError(f"port {q} has an empty terminal")
    fixed = np.unique(np.concatenate(plus + minus))
    fixed = np.unique(np.concatenate([fixed, floating_ground_nodes(lat, fixed)]))
    free = np.setdiff1d(np.arange(lat.M), fixed)
    Au, Ap = A[free], A[fixed]
    n5 = 5 * lat.K
    S = np.zeros((n5 + free.size, n5 + free.size), dtype=np.complex128)
    S[:n5, :n5] = Z
    S[:n5, n5:] = Au.T
    S[n5:, :n5] = Au
    P = len(ports)
    Y = np.zeros((P, P), dtype=np.complex128)
    fields = []
    lu_rhs = []
    for p in range(P):
        phi_p = np.isin(fixed, plus[p]).astype(np.float64)
        rhs = np.zeros(n5 + free.size, dtype=np.complex128)
        rhs[:n5] = -Ap.T @ phi_p
        lu_rhs.append(rhs)
    X = np.linalg.solve(S, np.stack(lu_rhs, 1))
    for p in range(P):
        I = X[:n5, p]
        flux = A @ I
        for q in range(P):
            Y[q, p] = -np.sum(flux[plus[q]])
        fields.append(dict(I=I, phi_free=X[n5:, p], kcl=Au @ I))
    Zp = np.linalg.inv(Y)
    res = dict(Y=Y, Z=Zp, L=Zp.imag / omega, R=Zp.real, free=free, fixed=fixed)
    if return_fields:
        res["fields"] = fields
    return res


def schur_preconditioner(lat: Lattice, materials, omega: float, dx: float, free):
    """Eq. 12-15 with an exact inverse of the Schur complement: Ybar = diag|Z_ii|
    (P:154), Sbar = Au Ybar^-1 Au^T factored by sparse LU (the LDL^T alternative the
    paper compares AGMG with).  Returns x -> Q^-1 x for the reduced saddle system
    [Z Au^T; Au 0] (reading G12 signs)."""
    import scipy.sparse.linalg as spla
    from . import kernels
    from .operator import MU0, local_terms
    A = lat.incidence().tocsr()
    Au = A[free]
    n5 = 5 * lat.K
    # |Z_ii| = |z^b + j w mu0 dx T^{bb}(0)|
    T0 = kernels.toeplitz_blocks(np.zeros((1, 3), dtype=np.int64))
    self_g = np.array([T0[(b, b)][0] for b in kernels.BASES])
    zl = local_terms(lat, materials, omega, dx)                  # (5, K)
    yd = np.abs(zl + 1j * omega * MU0 * dx * self_g[:, None]).ravel()
    yinv = 1.0 / yd
    Sb = (Au @ sp.diags(yinv) @ Au.T).tocsc()
    lu = spla.splu(Sb)

    def apply(x):
        # Eq. 13-15 for Eq. 7's [Z -A^T; A 0] (Phi_7 = -Phi here, reading G12):
        # e = d - A Y^-1 c,  b = S^-1 e,  a = Y^-1 (c + A^T b),  Phi = -b
        c, d = x[:n5], x[n5:]
        e = d - Au @ (yinv * c)
        b = lu.solve(np.ascontiguousarray(e.real)) + 1j * lu.solve(np.ascontiguousarray(e.imag))
        a = yinv * (c + Au.T @ b)
        return np.concatenate([a, -b])
    return apply


def solve_ports_iterative(lat: Lattice, materials, omega: float, dx: float, ports, rtol=1e-10, workers=1):
    """The same reduced saddle system as ``solve_ports`` (G12/G13/G14) solved by GMRES(50)
     with the Schur preconditioner of Eq. 12-15 (exact sparse inverse of Sbar) and the
    oracle's direct-sum product for Z (operator.matvec_direct): for grids too large for a dense
    solve (configs 2-3).  ``workers`` > 1 splits the direct sum over processes by output rows."""
    import scipy.sparse.linalg as spla
    from .operator import GreenTable, matvec_direct
    A = lat.incidence().tocsr()
    plus = [port_nodes(lat, p["plus"]) for p in ports]
    minus = [port_nodes(lat, p["minus"]) for p in ports]
    fixed = np.unique(np.concatenate(plus + minus))
    fixed = np.unique(np.concatenate([fixed, floating_ground_nodes(lat, fixed)]))
    free = np.setdiff1d(np.arange(lat.M), fixed)
    Au, Ap = A[free], A[fixed]
    n5 = 5 * lat.K
    n = n5 + free.size
    table = GreenTable(lat)
    chunks = np.array_split(np.arange(lat.K), max(1, workers))
    pool = None
    if workers > 1:
        import multiprocessing as mp
        global _POOL_STATE
        _POOL_STATE = (lat, materials, omega, dx, table)
        pool = mp.get_context("fork").Pool(workers)

    def zmul(I):
        I5 = I.reshape(5, lat.K)
        if pool is None:
            return matvec_direct(lat, materials, omega, dx, I5, table=table).ravel()
        parts = pool.starmap(_zmul_rows, [(I5, r) for r in chunks])
        out = np.zeros((5, lat.K), dtype=np.complex128)
        for r, p in zip(chunks, parts):
            out[:, r] = p
        return out.ravel()

    def sysmul(x):
        y = np.empty(n, dtype=np.complex128)
        y[:n5] = zmul(x[:n5]) + Au.T @ x[n5:]
        y[n5:] = Au @ x[:n5]
        return y

    Aop = spla.LinearOperator((n, n), matvec=sysmul, dtype=np.complex128)
    Mop = spla.LinearOperator((n, n), matvec=schur_preconditioner(lat, materials, omega, dx, free),
                              dtype=np.complex128)
    P = len(ports)
    Y = np.zeros((P, P), dtype=np.complex128)
    info = []
    for p in range(P):
        phi_p = np.isin(fixed, plus[p]).astype(np.float64)
        rhs = np.zeros(n, dtype=np.complex128)
        rhs[:n5] = -Ap.T @ phi_p
        x, code = spla.gmres(Aop, rhs, M=Mop, rtol=rtol, atol=0.0, restart=50, maxiter=200)
        res = np.linalg.norm(rhs - sysmul(x)) / np.linalg.norm(rhs)
        info.append(dict(code=int(code), rre=float(res)))
        flux = A @ x[:n5]
        for q in range(P):
            Y[q, p] = -np.sum(flux[plus[q]])
    if pool is not None:
        pool.close()
    Zp = np.linalg.inv(Y)
    return dict(Y=Y, Z=Zp, L=Zp.imag / omega, R=Zp.real, info=info)


_POOL_STATE = None


def _zmul_rows(I5, rows):
    from .operator import matvec_direct
    lat, materials, omega, dx, table = _POOL_STATE
    return matvec_direct(lat, materials, omega, dx, I5, rows=rows, table=table)
