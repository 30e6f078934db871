"""Oracle: the SuperVoxHenry impedance operator Z (Eq. 8) and its product Z.I.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The method (Eq. 9) computes CC = Z.I with FFTs of circulant
embeddings.  That is exactly (up to rounding) the dense product with
  Z^{b,a}_{lk} = delta_lk delta_ba z^b_l + jw mu0 dx T^{b,a}(r_l - r_k)
(App. A; G1 basis normalisation, see kernels.py), so the
oracle is that product written out: a direct sum over voxel pairs.  No FFT,
no circulant, no symmetry shortcut.

Local (diagonal) term, App. A Eq. 16-18 and P:83:
  z^b = c / (w_b dx),  w = (1, 1, 1, 6, 2) for (x, y, z, 2D, 3D),
  c = a + j w mu b,  a, b from Eq. 22-23 (two-fluid conductivity Eq. 3).
mu = mu0 = 4 pi 1e-7 H/m (reading G4).  omega = 2 pi f (G21).
A material with lambda = inf is a normal conductor: Eq. 22-23 in the limit
lambda -> inf give a = 1/sigma0, b = 0 (reading G5).
"""
from __future__ import annotations

import numpy as np

from . import kernels
from .lattice import Lattice

MU0 = 4e-7 * np.pi
BASES = kernels.BASES
LOCAL_DIVISOR = {"x": 1.0, "y": 1.0, "z": 1.0, "2D": 6.0, "3D": 2.0}


def two_fluid_sigma(sigma0, lam, omega):
    """Eq. 3: sigma = sigma0 - j/(w mu lambda^2)."""
    lam = np.asarray(lam, dtype=np.float64)
    with np.errstate(divide="ignore"):
        sup = np.where(np.isinf(lam), 0.0, 1.0 / (omega * MU0 * lam ** 2))
    return np.asarray(sigma0, dtype=np.float64) - 1j * sup


def two_fluid_ab(sigma0, lam, omega):
    """Eq. 22-23: a = s0 (w mu l^2)^2 / (1 + (s0 w mu l^2)^2), b = l^2 / (1 + (s0 w mu l^2)^2).

    lambda = inf (normal conductor): limit a -> 1/sigma0, b -> 0.
    """
    sigma0 = np.asarray(sigma0, dtype=np.float64)
    lam = np.asarray(lam, dtype=np.float64)
    if np.isinf(lam).any():
        if (np.isinf(lam) & (sigma0 <= 0)).any():
            raise ValueError("lambda = inf requires sigma0 > 0")
    inf = np.isinf(lam)
    lam_f = np.where(inf, 1.0, lam)
    g = omega * MU0 * lam_f ** 2
    den = 1.0 + (sigma0 * g) ** 2
    a = np.where(inf, 1.0 / np.where(sigma0 > 0, sigma0, 1.0), sigma0 * g ** 2 / den)
    b = np.where(inf, 0.0, lam_f ** 2 / den)
    return a, b


def local_terms(lat: Lattice, materials, omega: float, dx: float):
    """z^b_l for every voxel: array (5, K) complex, component-major."""
    mats = np.asarray(materials, dtype=np.float64).reshape(-1, 2)
    s0 = mats[lat.voxel_mat - 1, 0]
    lm = mats[lat.voxel_mat - 1, 1]
    a, b = two_fluid_ab(s0, lm, omega)
    c = a + 1j * omega * MU0 * b
    return np.stack([c / (LOCAL_DIVISOR[bn] * dx) for bn in BASES])


class GreenTable:
    """T^{b,a}(m) on the full signed offset box of a lattice (tiny / mid grids)."""

    def __init__(self, lat: Lattice):
        self.ext = np.array([lat.Kx, lat.Ky, lat.Kz])
        rng = [np.arange(-(e - 1), e) for e in self.ext]
        MX, MY, MZ = np.meshgrid(*rng, indexing="ij")
        offs = np.stack([MX.ravel(), MY.ravel(), MZ.ravel()], axis=1)
        self.shape = tuple(2 * self.ext - 1)
        self.blocks = kernels.toeplitz_blocks(offs)  # unit voxel

    def lookup(self, offs):
        """Flat index of offsets (..., 3) into the table."""
        o = offs + (self.ext - 1)
        return (o[..., 0] * self.shape[1] + o[..., 1]) * self.shape[2] + o[..., 2]


class SampledGreen:
    """T^{b,a}(m) computed only at the offsets a given set of rows needs (large grids)."""

    def __init__(self, lat: Lattice, rows):
        offs = (lat.coords[np.asarray(rows)][:, None, :] - lat.coords[None, :, :]).reshape(-1, 3)
        self.uniq, self.inv = np.unique(offs, axis=0, return_inverse=True)
        self.inv = self.inv.reshape(len(rows), lat.K)
        self.blocks = kernels.toeplitz_blocks(self.uniq)


def dense_Z(lat: Lattice, materials, omega: float, dx: float, green_only: bool = False):
    """Dense 5K x 5K complex Z (Eq. 8) for tiny grids."""
    K = lat.K
    offs = lat.coords[:, None, :] - lat.coords[None, :, :]
    T = kernels.toeplitz_blocks(offs.reshape(-1, 3))
    Z = np.zeros((5 * K, 5 * K), dtype=np.complex128)
    pref = 1j * omega * MU0 * dx
    for bi, b in enumerate(BASES):
        for ai, a in enumerate(BASES):
            Z[bi * K:(bi + 1) * K, ai * K:(ai + 1) * K] = pref * T[(b, a)].reshape(K, K)
    if not green_only:
        z = local_terms(lat, materials, omega, dx)
        Z[np.arange(5 * K), np.arange(5 * K)] += z.ravel()
    return Z


def matvec_direct(lat: Lattice, materials, omega: float, dx: float, I, green_only=False,
                  rows=None, table=None, chunk=64):
    """Direct-sum CC = Z.I for I of shape (5, K) (or (nrhs, 5, K)).

    rows: optional subset of observation voxels (indices into 0..K-1); the
    result then has shape (..., 5, len(rows)).  The Green sum runs over every
    source voxel k: CC^b_l = z^b_l I^b_l + jw mu0 dx sum_a sum_k T^{b,a}(r_l - r_k) I^a_k.
    """
    I = np.asarray(I, dtype=np.complex128)
    single = I.ndim == 2
    if single:
        I = I[None]
    K = lat.K
    rows = np.arange(K) if rows is None else np.asarray(rows)
    pref = 1j * omega * MU0 * dx
    out = np.zeros((I.shape[0], 5, rows.size), dtype=np.complex128)
    if table is None:
        table = SampledGreen(lat, rows) if rows.size < K else GreenTable(lat)
    for c0 in range(0, rows.size, chunk):
        rr = rows[c0:c0 + chunk]
        if isinstance(table, SampledGreen):
            idx = table.inv[c0:c0 + chunk]
        else:
            idx = table.lookup(lat.coords[rr][:, None, :] - lat.coords[None, :, :])
        for bi, b in enumerate(BASES):
            acc = np.zeros((I.shape[0], rr.size), dtype=np.complex128)
            for ai, a in enumerate(BASES):
                tb = table.blocks[(b, a)]
                if not np.any(tb):
                    continue
                acc += np.einsum("lk,rk->rl", tb[idx], I[:, ai, :])
            out[:, bi, c0:c0 + chunk] = pref * acc
    if not green_only:
        z = local_terms(lat, materials, omega, dx)
        out += z[None, :, rows] * I[:, :, rows]
    return out[0] if single else out
