"""Pins for oracle/operator.py and oracle/lattice.py (CPU only)."""
import numpy as np
import pytest
from scipy import signal

import svh_inputs
from oracle import kernels
from oracle.lattice import Lattice
from oracle.operator import (MU0, GreenTable, dense_Z, local_terms, matvec_direct,
                             two_fluid_ab, two_fluid_sigma)


def test_two_fluid_c_is_inverse_sigma():
    """Eq. 22-23 vs Eq. 3: c = a + j w mu b equals 1/sigma exactly (reading G5)."""
    g = np.random.default_rng(0)
    s0 = g.uniform(0, 5e7, 50)
    lam = g.uniform(20e-9, 2e-6, 50)
    w = 2 * np.pi * g.uniform(1e8, 1e11, 50)
    for i in range(50):
        a, b = two_fluid_ab(s0[i], lam[i], w[i])
        c = a + 1j * w[i] * MU0 * b
        assert abs(c * two_fluid_sigma(s0[i], lam[i], w[i]) - 1) < 1e-14


def test_two_fluid_limits():
    """SPEC kernels examples: sigma0 = 0 -> a = 0, b = lambda^2; unit product -> halves;
    lambda = inf -> normal conductor a = 1/sigma0, b = 0 (reading G5)."""
    a, b = two_fluid_ab(0.0, 90e-9, 2 * np.pi * 1e10)
    assert a == 0 and abs(b - (90e-9) ** 2) < 1e-30
    lam = 1e-7
    w = 2 * np.pi * 1e10
    s0 = 1.0 / (w * MU0 * lam ** 2)
    a, b = two_fluid_ab(s0, lam, w)
    assert np.isclose(a, s0 * (w * MU0 * lam ** 2) ** 2 / 2, rtol=1e-14)
    assert np.isclose(b, lam ** 2 / 2, rtol=1e-14)
    a, b = two_fluid_ab(1.7e7, np.inf, w)
    assert np.isclose(a, 1 / 1.7e7, rtol=1e-15) and b == 0
    a2, b2 = two_fluid_ab(1.7e7, 1e3, w)  # large finite lambda approaches the limit
    assert np.isclose(a2, 1 / 1.7e7, rtol=1e-9)


def test_local_term_ratios():
    """P7: z^2D / z^x = 1/6, z^3D / z^x = 1/2, sigma0 = 0 => imaginary, halving dx doubles |z|."""
    lat = Lattice(np.ones((1, 1, 3), np.uint8))
    z = local_terms(lat, [(0.0, 90e-9)], 2 * np.pi * 1e10, 0.25e-6)
    assert np.allclose(z[3] / z[0], 1 / 6) and np.allclose(z[4] / z[0], 1 / 2)
    assert np.allclose(z[0], z[1]) and np.allclose(z[0], z[2])
    assert np.all(z.real == 0)
    z2 = local_terms(lat, [(0.0, 90e-9)], 2 * np.pi * 1e10, 0.125e-6)
    assert np.allclose(np.abs(z2), 2 * np.abs(z))


def test_lattice_counts():
    """P14 / SPEC voxgrid: 1x1x1 -> K=1, M=6, N=11; 2x1x1 -> K=2, M=11, N=21."""
    for shape, (K, M) in [((1, 1, 1), (1, 6)), ((1, 1, 2), (2, 11)), ((2, 2, 2), (8, 36))]:
        lat = Lattice(np.ones(shape, np.uint8))
        assert (lat.K, lat.M, lat.N) == (K, M, 5 * K + M)


def test_incidence_flux_by_divergence_theorem():
    """Each A entry equals the outward flux of Eq. 4-6 through that face (face GL
    quadrature of f.n, G1 normalisation, dx=1), and every column sums to 0 (div f = 0)."""
    m = svh_inputs.random_fill((4, 3, 2), fill=0.6, seed=11)["mat_id"]
    lat = Lattice(m)
    A = lat.incidence().toarray()
    assert np.allclose(A.sum(0), 0)
    x, w = np.polynomial.legendre.leggauss(4)
    x = x / 2
    w = w / 2
    U, V = np.meshgrid(x, x, indexing="ij")
    WW = np.outer(w, w).ravel()

    def field(name, d):
        f = np.zeros_like(d)
        if name in ("x", "y", "z"):
            f[:, "xyz".index(name)] = 1
        elif name == "2D":
            f[:, 0], f[:, 1] = d[:, 0], -d[:, 1]
        else:
            f[:, 0], f[:, 1], f[:, 2] = d[:, 0], d[:, 1], -2 * d[:, 2]
        return f
    for k in range(lat.K):
        for bi, b in enumerate(kernels.BASES):
            col = A[:, bi * lat.K + k]
            for axis in range(3):
                for side in (-1, 1):
                    d = np.zeros((U.size, 3))
                    o = [q for q in range(3) if q != axis]
                    d[:, axis] = side * 0.5
                    d[:, o[0]], d[:, o[1]] = U.ravel(), V.ravel()
                    flux = np.sum(WW * field(b, d)[:, axis] * side)
                    node = lat.face_node(axis, lat.coords[k], side)
                    # the node row may also hold the neighbour's contribution to a
                    # different column; this column's entry is this voxel's flux only
                    assert abs(col[node] - flux) < 1e-14


def _case(shape, seed, n_mat=2):
    c = svh_inputs.random_fill(shape, fill=0.55, seed=seed, n_mat=n_mat)
    return Lattice(c["mat_id"]), c


def test_dense_symmetric_and_spd():
    """P4/P11/P12: Z is complex symmetric; for sigma0 = 0, Z/(jw) is real SPD."""
    lat, c = _case((3, 3, 2), 1)
    w = 2 * np.pi * c["freq"]
    Z = dense_Z(lat, c["materials"], w, c["dx"])
    assert np.allclose(Z, Z.T, rtol=0, atol=1e-14 * np.abs(Z).max())
    mats = [(0.0, 90e-9), (0.0, 200e-9)]
    Z0 = dense_Z(lat, mats, w, c["dx"]) / (1j * w)
    assert np.abs(Z0.imag).max() < 1e-14 * np.abs(Z0).max()
    ev = np.linalg.eigvalsh(Z0.real)
    assert ev.min() > 0


def test_direct_sum_matches_dense():
    lat, c = _case((4, 3, 3), 2)
    w = 2 * np.pi * c["freq"]
    I = svh_inputs.currents(lat.K, 2, seed=3)
    Z = dense_Z(lat, c["materials"], w, c["dx"])
    ref = np.einsum("ij,rj->ri", Z, I.reshape(2, -1)).reshape(2, 5, lat.K)
    got = matvec_direct(lat, c["materials"], w, c["dx"], I)
    assert np.allclose(got, ref, rtol=0, atol=1e-12 * np.abs(ref).max())
    rows = np.array([0, 5, lat.K - 1])
    sub = matvec_direct(lat, c["materials"], w, c["dx"], I, rows=rows)
    assert np.allclose(sub, ref[:, :, rows], rtol=0, atol=1e-12 * np.abs(ref).max())


def test_green_part_is_linear_convolution():
    """P17: the Green part equals scipy.signal.convolve(method='direct') of each
    zero-filled current grid with the signed-offset kernel (catches l-k vs k-l)."""
    lat, c = _case((5, 4, 3), 4)
    w = 2 * np.pi * c["freq"]
    I = svh_inputs.currents(lat.K, 1, seed=9)[0]
    got = matvec_direct(lat, c["materials"], w, c["dx"], I, green_only=True)
    tab = GreenTable(lat)
    shp = (lat.Kx, lat.Ky, lat.Kz)
    pref = 1j * w * MU0 * c["dx"]
    for bi, b in enumerate(kernels.BASES):
        acc = np.zeros(tuple(3 * np.array(shp) - 2), dtype=complex)
        for ai, a in enumerate(kernels.BASES):
            g = np.zeros(shp, dtype=complex)
            g[lat.coords[:, 0], lat.coords[:, 1], lat.coords[:, 2]] = I[ai]
            kern = tab.blocks[(b, a)].reshape(tab.shape)  # index offset + (K-1)
            acc += signal.convolve(g, kern, mode="full", method="direct")
        # full conv index n corresponds to offset n - (K-1) from source 0 => observation n-(K-1)
        crop = acc[lat.Kx - 1:2 * lat.Kx - 1, lat.Ky - 1:2 * lat.Ky - 1, lat.Kz - 1:2 * lat.Kz - 1]
        ref = pref * crop[lat.coords[:, 0], lat.coords[:, 1], lat.coords[:, 2]]
        assert np.allclose(got[bi], ref, rtol=0, atol=1e-12 * np.abs(ref).max())
