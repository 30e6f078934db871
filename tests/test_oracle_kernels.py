"""Pins for oracle/kernels.py (CPU only).

Each pin checks the oracle against something other than itself: a closed
form, a brute-force 6-D integral written independently from Eq. 4-6, an
independent adaptive quadrature of a box integral, multipole asymptotes, or
symmetry identities.  Citations: PAPER.md lines (P:n).
"""
import numpy as np
import pytest

from oracle import kernels

from _pins import box_integral

FOUR_PI = 4 * np.pi


# ---------------------------------------------------------------- helpers
def basis_field(name, r, center, dx):
    """Eq. 4-6 written directly at absolute coordinates, G1 normalisation
    (PWC 1/dx^2, PWL 1/dx^3 so that currents are in amperes)."""
    d = r - center
    out = np.zeros_like(r)
    if name in ("x", "y", "z"):
        out[:, "xyz".index(name)] = 1.0 / dx ** 2
    elif name == "2D":
        out[:, 0] = d[:, 0] / dx ** 3
        out[:, 1] = -d[:, 1] / dx ** 3
    elif name == "3D":
        out[:, 0] = d[:, 0] / dx ** 3
        out[:, 1] = d[:, 1] / dx ** 3
        out[:, 2] = -2.0 * d[:, 2] / dx ** 3
    return out


def cube_rule(corner, dx, n):
    x, w = np.polynomial.legendre.leggauss(n)
    x = (x + 1) / 2 * dx
    w = w / 2 * dx
    X, Y, Z = np.meshgrid(x, x, x, indexing="ij")
    W = (w[:, None, None] * w[None, :, None] * w[None, None, :]).ravel()
    pts = np.stack([X.ravel(), Y.ravel(), Z.ravel()], 1) + np.asarray(corner, float)
    return pts, W


def brute_6d(beta, alpha, cell_l, cell_k, dx, n=10):
    """int_{V_l} int_{V_k} f^beta_l(r) . f^alpha_k(r') / (4 pi |r - r'|) by 6-D tensor GL."""
    cl = np.asarray(cell_l, float) * dx
    ck = np.asarray(cell_k, float) * dx
    rl, wl = cube_rule(cl, dx, n)
    rk, wk = cube_rule(ck, dx, n)
    fb = basis_field(beta, rl, cl + dx / 2, dx)
    fa = basis_field(alpha, rk, ck + dx / 2, dx)
    dot = fb @ fa.T
    dist = np.sqrt(((rl[:, None, :] - rk[None, :, :]) ** 2).sum(-1))
    return float(np.einsum("i,ij,j->", wl, dot / (FOUR_PI * dist), wk))


# ---------------------------------------------------------------- pins
@pytest.mark.parametrize("a,b", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_overlap_weight_matches_definition(a, b):
    """W_ab(s) = int p_a(u) p_b(u-s) du (definition) by 1-D GL on the overlap."""
    prof = [lambda u: np.ones_like(u), lambda u: u]
    for s in np.linspace(-1.2, 1.2, 37):
        lo, hi = max(-0.5, s - 0.5), min(0.5, s + 0.5)
        if hi <= lo:
            ref = 0.0
        else:
            x, w = np.polynomial.legendre.leggauss(8)
            u = lo + (x + 1) / 2 * (hi - lo)
            ref = np.sum(w * (hi - lo) / 2 * prof[a](u) * prof[b](u - s))
        assert abs(kernels.overlap_weight(a, b, s) - ref) < 1e-15


def test_self_term_closed_form():
    """P1: 4 pi K0(0) = mean inverse distance of two points in a unit cube (closed form)."""
    closed = ((2 / 5) * (1 + np.sqrt(2) - 2 * np.sqrt(3)) - 2 * np.pi / 3
              + 2 * np.log(1 + np.sqrt(2)) + 4 * np.log((1 + np.sqrt(3)) / np.sqrt(2)))
    k0 = kernels.seven_kernels([[0, 0, 0]])[0, 0]
    assert abs(FOUR_PI * k0 - closed) < 1e-13 * closed


SEPARATED = [(2, 1, 1), (-3, 2, 0), (0, -2, 3), (4, 0, -1), (1, -2, 0)]


@pytest.mark.parametrize("m", SEPARATED)
def test_blocks_vs_bruteforce_6d(m):
    """Every (beta, alpha) block vs a 6-D integral of Eq. 4-6 at absolute positions.

    Catches a wrong sign, a transposed block, a wrong W or an l-k / k-l mixup.
    Also pins the dx scaling (App. B): evaluated at dx = 2.5e-7 m.
    """
    dx = 2.5e-7
    cell_k = np.array([3, 5, 4])
    cell_l = cell_k + np.array(m)
    T = kernels.toeplitz_blocks([m], dx=dx)
    scale = abs(T[("x", "x")][0])
    for b in kernels.BASES:
        for a in kernels.BASES:
            ref = brute_6d(b, a, cell_l, cell_k, dx, n=10)
            assert abs(T[(b, a)][0] - ref) <= 1e-9 * scale, (b, a, T[(b, a)][0], ref)


@pytest.mark.parametrize("m", [(1, 1, 1), (1, 1, 0)])
def test_blocks_vs_bruteforce_touching(m):
    """Touching voxels (corner / edge contact): 6-D GL with 2x2x2 sub-cells, looser bound."""
    dx = 1.0
    T = kernels.toeplitz_blocks([m], dx=dx)
    scale = abs(T[("x", "x")][0])
    cell_k = np.zeros(3)
    cell_l = np.asarray(m, float)
    for b, a in [("x", "x"), ("x", "2D"), ("2D", "y"), ("3D", "3D"), ("3D", "z"), ("2D", "3D")]:
        # split each cube into 8 half-cells (basis centres stay at the full-voxel centre)
        tot = 0.0
        x, w = np.polynomial.legendre.leggauss(12)
        for ol in np.ndindex(2, 2, 2):
            for ok in np.ndindex(2, 2, 2):
                rl, wl = cube_rule(cell_l + 0.5 * np.array(ol), 0.5, 12)
                rk, wk = cube_rule(cell_k + 0.5 * np.array(ok), 0.5, 12)
                fb = basis_field(b, rl, cell_l + 0.5, dx)
                fa = basis_field(a, rk, cell_k + 0.5, dx)
                dist = np.sqrt(((rl[:, None, :] - rk[None, :, :]) ** 2).sum(-1))
                tot += np.einsum("i,ij,j->", wl, (fb @ fa.T) / (FOUR_PI * dist), wk)
        assert abs(T[(b, a)][0] - tot) <= 2e-6 * scale, (b, a, T[(b, a)][0], tot)


def test_toeplitz_invariance():
    """P4 / P:77-79: the entry depends only on r_l - r_k (two absolute placements)."""
    m = np.array([2, -1, 1])
    for b, a in [("x", "2D"), ("3D", "y"), ("2D", "2D")]:
        v1 = brute_6d(b, a, np.array([0, 3, 0]) + m, np.array([0, 3, 0]), 1.0, n=8)
        v2 = brute_6d(b, a, np.array([7, 1, 5]) + m, np.array([7, 1, 5]), 1.0, n=8)
        assert abs(v1 - v2) < 1e-13
        assert abs(kernels.toeplitz_blocks([m])[(b, a)][0] - v1) < 1e-8 * 0.05


@pytest.mark.parametrize("dims", [(2, 1, 1), (2, 2, 1), (2, 2, 2), (16, 2, 2), (5, 3, 1)])
def test_box_sum_rule(dims):
    """P5: sum_{l,k in box} K0(l - k) = (1/4pi) int int_{box^2} 1/|r-r'| (Hoer-Love box)."""
    a, b, c = dims
    cells = np.array(list(np.ndindex(a, b, c)))
    offs = (cells[:, None, :] - cells[None, :, :]).reshape(-1, 3)
    uniq, cnt = np.unique(offs, axis=0, return_counts=True)
    k0 = kernels.toeplitz_blocks(uniq)[("x", "x")]
    s = float(np.sum(cnt * k0))
    ref = box_integral(a, b, c)
    assert abs(s - ref) <= 1e-10 * ref, (s, ref)


def test_far_field_asymptotes():
    """P3: K0 -> 1/(4 pi |m|), K1_x -> m_x/(48 pi |m|^3), K2_x -> -(3 m_x^2 - |m|^2)/(576 pi |m|^5).

    Moments of W_00, W_01, W_11 fix the leading multipole terms; the relative
    deviation must fall at least like |m|^-2 when |m| doubles.
    """
    def lead(m):
        m = np.asarray(m, float)
        r = np.linalg.norm(m)
        return np.array([1 / (FOUR_PI * r), m[0] / (48 * np.pi * r ** 3),
                         -(3 * m[0] ** 2 - r ** 2) / (576 * np.pi * r ** 5)])
    for direction in [(1, 0, 0), (2, 1, 0), (3, 1, 2)]:
        d = np.array(direction)
        errs = []
        for s in (6, 12):
            m = d * s
            K = kernels.seven_kernels([m])[0]
            got = np.array([K[0], K[1], K[4]])
            errs.append(np.abs(got / lead(m) - 1))
        errs = np.array(errs)
        assert np.all(errs[0] < 0.05)
        assert np.all(errs[1] <= errs[0] / 3.5 + 1e-12), errs


def test_parity_and_reciprocity():
    """P4: K0, K2 even on every axis; K1_c odd on c, even on others; T^{ba}(m) = T^{ab}(-m);
    the Eq. 8 zero blocks vanish; T^{xx} = T^{yy} = T^{zz} up to axis permutation."""
    rng = np.random.default_rng(1)
    ms = rng.integers(-4, 5, size=(12, 3))
    K = kernels.seven_kernels(ms)
    for ax in range(3):
        flip = ms.copy()
        flip[:, ax] *= -1
        Kf = kernels.seven_kernels(flip)
        assert np.allclose(Kf[:, 0], K[:, 0], rtol=1e-13, atol=1e-17)
        for c in range(3):
            sgn = -1 if c == ax else 1
            assert np.allclose(Kf[:, 1 + c], sgn * K[:, 1 + c], rtol=1e-12, atol=1e-17)
            assert np.allclose(Kf[:, 4 + c], K[:, 4 + c], rtol=1e-12, atol=1e-17)
    T = kernels.toeplitz_blocks(ms)
    Tm = kernels.toeplitz_blocks(-ms)
    for b in kernels.BASES:
        for a in kernels.BASES:
            assert np.allclose(T[(b, a)], Tm[(a, b)], rtol=1e-12, atol=1e-15)
    for b, a in [("x", "y"), ("x", "z"), ("y", "z"), ("z", "2D")]:
        assert not np.any(T[(b, a)]) and not np.any(T[(a, b)])
    perm = ms[:, [1, 0, 2]]
    assert np.allclose(kernels.toeplitz_blocks(perm)[("y", "y")], T[("x", "x")], rtol=1e-13)


def test_quadrature_converged():
    """Order schedule is converged: +6 GL orders change every reduced integral < 1e-12 of K0."""
    offs = np.array([[2, 0, 0], [2, 2, 1], [3, 1, 0], [5, 2, 2], [9, 0, 1], [15, 7, 3], [25, 3, 1]])
    base = kernels.reduced_integrals(offs)
    orders = kernels.far_order(offs)
    for i, m in enumerate(offs):
        ref = kernels.reduced_integrals([m], order=int(orders[i]) + 6)[0]
        assert np.max(np.abs(base[i] - ref)) < 1e-12 * abs(base[i][0]), (m, base[i] - ref)
    near = np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [1, 1, 1], [1, -1, 0]])
    a = kernels.reduced_integrals(near)
    b = kernels.reduced_integrals(near, n_duffy=28, n_near=28)
    assert np.max(np.abs(a - b)) < 1e-14


def test_dx5_law():
    """App. B Eq. 24-27: the un-normalised PWC integral at edge dx is dx^5 x (dx = 1)."""
    for dx in (2.0, 0.5):
        m = (2, 1, 0)
        # brute_6d includes the 1/dx^4 basis normalisation; multiply it back out
        v_dx = brute_6d("x", "x", np.array(m), np.zeros(3), dx, n=8) * dx ** 4
        v_1 = brute_6d("x", "x", np.array(m), np.zeros(3), 1.0, n=8)
        assert abs(v_dx - dx ** 5 * v_1) < 1e-12 * abs(v_dx)
