"""Oracle: Galerkin interaction integrals of the SuperVoxHenry voxel bases.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  fp64, numpy.

What the paper fixes
--------------------
* Bases per non-empty voxel k (Eq. 4-6): PWC f^x, f^y, f^z and PWL
  f^2D = ((x-x_k) x^ - (y-y_k) y^)/dx,  f^3D = ((x-x_k) x^ + (y-y_k) y^ - 2(z-z_k) z^)/dx.
* Galerkin testing of the Green term jw mu int G J (Eq. 1) with
  G = 1/(4 pi |r-r'|) gives entries jw mu int_l int_k f^b . G f^a
  (App. A P:301-321 for the self terms).
* The entries depend only on the voxel offset l-k: block Toeplitz tensors
  T^{b,a}.
* Scaling factor dx^5 (App. B, Eq. 24-27).

Readings taken
---------------------------------------------------------
* Basis normalisation G1: currents in amperes, i.e. f^x = x^/dx^2 and the PWL
  bases carry 1/dx^3.  With u = (r - r_k)/dx every basis is (1/dx^2) times a
  unit-voxel profile, so Z_green = jw mu0 dx * T(unit voxel).  T here is the
  unit-voxel (dx = 1) integral, exactly Appendix B's dx^5 law applied to the
  paper's 1/dx^4 (Eq. 16) prefactor.
* Sign G2: Eq. 19-21 print a leading minus; we take + (Eq. 1 has +jw mu int G J).
* Eq. 21 garbled G3: weights (x, y, 4z) follow from the Eq. 6 dot product,
  and in general every block is the dot product of the two basis vectors.

Reduction used (exact, not an approximation)
--------------------------------------------
Along one axis a unit-voxel basis component is a profile p_0(u) = 1 (PWC) or
p_1(u) = u (PWL), u in [-1/2, 1/2].  For a separable integrand
  int int p_a(u) p_b(u') g(u - u' + m) du du' = int W_ab(s) g(s + m) ds,
  W_ab(s) = int p_a(u) p_b(u - s) du   (over the overlap of the two voxels),
so every 6-D block integral is a 3-D integral over s in [-1,1]^3:
  K(m; W_x, W_y, W_z) = 1/(4 pi) int W_x(s_x) W_y(s_y) W_z(s_z) / |s + m| ds.
W_ab is written out in closed form in ``overlap_weight`` and checked against a
direct 1-D quadrature of its definition in tests (pin).  The reduced integrals
are evaluated on the 8 unit sub-cubes of [-1,1]^3 (the |s| kinks sit on their
faces): a sub-cube having the singular point s = -m as a vertex is Duffy-mapped
(3 pyramids, Jacobian u^2 cancels 1/r); every other sub-cube uses tensor
Gauss-Legendre whose order depends on its distance to -m.

Pins (tests/test_oracle_kernels.py): closed-form unit-cube self term (P1),
direct 6-D Gauss-Legendre of f^b.G f^a at absolute voxel positions (brute
force, checks every block, sign and the Toeplitz invariance), the box sum rule
via an independent adaptive 2-D quadrature (P5), far-field multipole limits
(P3), parity identities (P4) and the dx^5 law (P6).
"""
from __future__ import annotations

import functools
import itertools

import numpy as np

FOUR_PI = 4.0 * np.pi

# Component order of the unknown vector: I = [I^x; I^y; I^z; I^2D; I^3D]
BASES = ("x", "y", "z", "2D", "3D")

# Basis vectors of Eq. 4-6 at unit voxel, as a list of (axis, coefficient,
# (profile_x, profile_y, profile_z)); profile 0 = constant, 1 = linear u.
BASIS_COMPONENTS = {
    "x": [(0, 1.0, (0, 0, 0))],
    "y": [(1, 1.0, (0, 0, 0))],
    "z": [(2, 1.0, (0, 0, 0))],
    "2D": [(0, 1.0, (1, 0, 0)), (1, -1.0, (0, 1, 0))],            # Eq. 5
    "3D": [(0, 1.0, (1, 0, 0)), (1, 1.0, (0, 1, 0)), (2, -2.0, (0, 0, 1))],  # Eq. 6
}


def overlap_weight(a: int, b: int, s):
    """W_ab(s) = int p_a(u) p_b(u - s) du, u and u - s in [-1/2, 1/2].

    a = test profile, b = source profile; p_0 = 1, p_1 = u.  Closed forms
    (derivation: integrate the polynomial over the overlap interval):
      W_00 = 1 - |s|,  W_01 = -s (1 - |s|)/2,  W_10 = +s (1 - |s|)/2,
      W_11 = 1/12 - |s|/4 + |s|^3/6,   zero for |s| > 1.
    """
    s = np.asarray(s, dtype=np.float64)
    t = np.abs(s)
    inside = t <= 1.0
    if (a, b) == (0, 0):
        w = 1.0 - t
    elif (a, b) == (0, 1):
        w = -s * (1.0 - t) / 2.0
    elif (a, b) == (1, 0):
        w = s * (1.0 - t) / 2.0
    elif (a, b) == (1, 1):
        w = 1.0 / 12.0 - t / 4.0 + t ** 3 / 6.0
    else:
        raise ValueError((a, b))
    return np.where(inside, w, 0.0)


def block_terms(beta: str, alpha: str):
    """Expand f^beta . f^alpha' into separable terms.

    Returns a list of (coef, triple) where triple = ((a_x,b_x),(a_y,b_y),(a_z,b_z))
    are the (test, source) profile pairs per axis.  Only components along the
    same axis contribute (dot product).  Empty list = structurally zero block
    (Eq. 8 zeros: (x,y), (x,z), (y,z), (z,2D) and transposes).
    """
    terms = []
    for ax_b, c_b, p_b in BASIS_COMPONENTS[beta]:
        for ax_a, c_a, p_a in BASIS_COMPONENTS[alpha]:
            if ax_a != ax_b:
                continue
            triple = tuple((p_b[d], p_a[d]) for d in range(3))
            terms.append((c_b * c_a, triple))
    return terms


@functools.lru_cache(maxsize=None)
def all_triples():
    s = set()
    for b in BASES:
        for a in BASES:
            for _, tr in block_terms(b, a):
                s.add(tr)
    return tuple(sorted(s))


# ----------------------------------------------------------------------------
# quadrature rules on [0,1]
@functools.lru_cache(maxsize=None)
def _gl01(n: int):
    x, w = np.polynomial.legendre.leggauss(n)
    return 0.5 * (x + 1.0), 0.5 * w


_SUBCUBES = list(itertools.product((-1.0, 0.0), repeat=3))  # lower corners


@functools.lru_cache(maxsize=None)
def _plain_rule(n: int):
    """Tensor GL of order n on each of the 8 unit sub-cubes of [-1,1]^3."""
    x, w = _gl01(n)
    X, Y, Z = np.meshgrid(x, x, x, indexing="ij")
    Wt = (w[:, None, None] * w[None, :, None] * w[None, None, :]).ravel()
    base = np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1)
    pts, wts = [], []
    for c in _SUBCUBES:
        pts.append(base + np.asarray(c))
        wts.append(Wt)
    return np.concatenate(pts), np.concatenate(wts)


@functools.lru_cache(maxsize=None)
def _duffy_unit(n: int):
    """Duffy rule on [0,1]^3 for an integrand singular (1/r) at the origin.

    The cube is split into the 3 pyramids {t_i = max_j t_j}; each is the image
    of [0,1]^3 under (u,v,w) -> u * (e_i + v e_j + w e_k), Jacobian u^2.
    Returns points t (P x 3) and weights.
    """
    x, w = _gl01(n)
    U, V, W = np.meshgrid(x, x, x, indexing="ij")
    WU, WV, WW = np.meshgrid(w, w, w, indexing="ij")
    U, V, W = U.ravel(), V.ravel(), W.ravel()
    jac = (WU * WV * WW).ravel() * U ** 2
    pts, wts = [], []
    for i in range(3):
        j, k = [d for d in range(3) if d != i]
        t = np.empty((U.size, 3))
        t[:, i] = U
        t[:, j] = U * V
        t[:, k] = U * W
        pts.append(t)
        wts.append(jac)
    return np.concatenate(pts), np.concatenate(wts)


def _near_rule(m, n_duffy: int, n_plain: int):
    """Quadrature rule over [-1,1]^3 for an offset with -m inside the cube."""
    p = -np.asarray(m, dtype=np.float64)
    xg, wg = _gl01(n_plain)
    X, Y, Z = np.meshgrid(xg, xg, xg, indexing="ij")
    base = np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1)
    Wb = (wg[:, None, None] * wg[None, :, None] * wg[None, None, :]).ravel()
    tpts, twts = _duffy_unit(n_duffy)
    pts, wts = [], []
    for c in _SUBCUBES:
        lo = np.asarray(c)
        hi = lo + 1.0
        is_vertex = np.all((p == lo) | (p == hi))
        if is_vertex:
            # map t in [0,1]^3 (singular at t=0) onto the sub-cube with t=0 at p
            sign = np.where(p == lo, 1.0, -1.0)
            pts.append(p + sign * tpts)
            wts.append(twts)
        else:
            pts.append(base + lo)
            wts.append(Wb)
    return np.concatenate(pts), np.concatenate(wts)


def _weight_matrix(pts, wts, triples):
    cols = []
    for (ax, bx), (ay, by), (az, bz) in triples:
        cols.append(wts * overlap_weight(ax, bx, pts[:, 0])
                    * overlap_weight(ay, by, pts[:, 1])
                    * overlap_weight(az, bz, pts[:, 2]))
    return np.stack(cols, axis=1)


def far_order(m) -> int:
    """GL order per sub-cube axis for |m|_inf >= 2, by distance of -m to [-1,1]^3.

    Orders chosen so that a +6 order increase changes every reduced integral
    by < 1e-13 relative (checked in tests/test_oracle_kernels.py).
    """
    m = np.abs(np.asarray(m, dtype=np.float64))
    d = np.sqrt(np.sum(np.maximum(m - 1.0, 0.0) ** 2, axis=-1))
    return np.where(d < 1.5, 16, np.where(d < 3.5, 12, np.where(d < 8.0, 9, np.where(d < 20.0, 7, 5))))


def reduced_integrals(offsets, triples=None, n_duffy: int = 20, n_near: int = 20, order=None):
    """K(m; triple) for every offset m (integer, shape (P,3)) and triple.

    Returns array (P, len(triples)).  ``order`` overrides the far-field GL
    order (used by the convergence pin).
    """
    if triples is None:
        triples = all_triples()
    offs = np.atleast_2d(np.asarray(offsets, dtype=np.float64))
    out = np.empty((offs.shape[0], len(triples)))
    near = np.max(np.abs(offs), axis=1) <= 1.0
    for idx in np.nonzero(near)[0]:
        pts, wts = _near_rule(offs[idx], n_duffy, n_near)
        WT = _weight_matrix(pts, wts, triples)
        r = np.sqrt(np.sum((pts + offs[idx]) ** 2, axis=1))
        out[idx] = (1.0 / r) @ WT / FOUR_PI
    far_idx = np.nonzero(~near)[0]
    if far_idx.size:
        orders = far_order(offs[far_idx]) if order is None else np.full(far_idx.size, order)
        for n in np.unique(orders):
            sel = far_idx[orders == n]
            pts, wts = _plain_rule(int(n))
            WT = _weight_matrix(pts, wts, triples)
            chunk = max(1, int(4e6 // pts.shape[0]))
            for c0 in range(0, sel.size, chunk):
                ii = sel[c0:c0 + chunk]
                d = pts[None, :, :] + offs[ii][:, None, :]
                r = np.sqrt(np.einsum("pqk,pqk->pq", d, d))
                out[ii] = (1.0 / r) @ WT / FOUR_PI
    return out


def toeplitz_blocks(offsets, dx: float = 1.0):
    """T^{b,a}(m) for all 25 (b,a) pairs at offsets m = l - k (observation minus source).

    Returns dict {(beta, alpha): array (P,)} of the Galerkin integral
    int_l int_k f^b(r) . f^a(r') / (4 pi |r - r'|) dV' dV with the G1 basis
    normalisation.  dx != 1 evaluates the physical-size integral, which
    equals dx * T(unit) for G1-normalised bases (dx^5 law with the
    1/dx^4 basis normalisation).  Structurally zero blocks are exact zeros.
    """
    triples = all_triples()
    R = reduced_integrals(offsets, triples)
    col = {t: i for i, t in enumerate(triples)}
    res = {}
    for b in BASES:
        for a in BASES:
            v = np.zeros(R.shape[0])
            for coef, tr in block_terms(b, a):
                v = v + coef * R[:, col[tr]]
            res[(b, a)] = v * dx
    return res


def seven_kernels(offsets):
    """The 7 distinct unit-voxel kernels named in SURVEY 8(c):
    K0, K1_x, K1_y, K1_z, K2_x, K2_y, K2_z (each = K(m; W..) with one non-W_00 axis).

    K1_c uses W_01 (PWC test, PWL source) on axis c, K2_c uses W_11 on axis c.
    Returned as (P, 7).  Used to state DESIGN.md's kernel table; T^{b,a} are
    built from block_terms, not from this table.
    """
    z = (0, 0)
    trip = [(z, z, z)]
    for c in range(3):
        t = [z, z, z]
        t[c] = (0, 1)
        trip.append(tuple(t))
    for c in range(3):
        t = [z, z, z]
        t[c] = (1, 1)
        trip.append(tuple(t))
    return reduced_integrals(offsets, tuple(trip))
