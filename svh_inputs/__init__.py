"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method: only voxel geometries
(material-id arrays), material tables, port face sets and seeded random
current vectors.  The recipes follow SURVEY.md 8(d) ("Configs restated as
concrete synthetic inputs") and BASELINE.json ``configs``; the paper's own
layouts and measurement data are not available, so every geometry here is a
synthetic stand-in with the paper's workload shape (thin superconducting films
over ground planes P:178, a sharp bend P:234, a multilayer eSFQ-like
subsystem P:266).  DESIGN.md "Input recipe" restates them.

Conventions (identical to include/svh.h):
* ``mat_id``: uint8 array of shape (Kz, Ky, Kx) (x fastest); 0 = empty voxel,
  m >= 1 indexes ``materials[m-1] = (sigma0 [S/m], lambda_L [m])``;
  lambda_L = inf marks a normal conductor.
* A port is ``{"plus": [face_rect...], "minus": [face_rect...]}`` with
  ``face_rect = (axis, side, lo_xyz, hi_xyz)``: the faces on ``side`` (-1/+1)
  of ``axis`` (0=x,1=y,2=z) of every voxel in the half-open box [lo, hi).
* Random currents: i.i.d. complex normal (re, im ~ N(0,1)), numpy PCG64.
"""
from __future__ import annotations

import numpy as np

NB = (1.7e7, 90e-9)   # Nb-like two-fluid material used by configs 1-4 (BASELINE.json)


def rng(seed):
    return np.random.Generator(np.random.PCG64(seed))


def currents(K: int, nrhs: int = 1, seed: int = 0, dtype=np.complex128):
    """(nrhs, 5, K) i.i.d. complex normal current coefficients."""
    g = rng(seed)
    re = g.standard_normal((nrhs, 5, K))
    im = g.standard_normal((nrhs, 5, K))
    return (re + 1j * im).astype(dtype)


def _box(mat, lo, hi, val=1):
    (x0, y0, z0), (x1, y1, z1) = lo, hi
    mat[z0:z1, y0:y1, x0:x1] = val


def config1():
    """BASELINE configs[0]: straight Nb bar 16x2x2, dx 0.25 um, f 10 GHz, end-face port."""
    mat = np.ones((2, 2, 16), dtype=np.uint8)
    port = {"plus": [(0, +1, (15, 0, 0), (16, 2, 2))], "minus": [(0, -1, (0, 0, 0), (1, 2, 2))]}
    return dict(name="cfg1_bar_16x2x2", mat_id=mat, dx=0.25e-6, materials=[NB], freq=10e9,
                ports=[port])


def bar(n, ny=1, nz=1, dx=0.25e-6, material=NB, freq=10e9):
    """n x ny x nz bar with end-face port (pin variants P8-P10 of SURVEY 8(c))."""
    mat = np.ones((nz, ny, n), dtype=np.uint8)
    port = {"plus": [(0, +1, (n - 1, 0, 0), (n, ny, nz))], "minus": [(0, -1, (0, 0, 0), (1, ny, nz))]}
    return dict(name=f"bar_{n}x{ny}x{nz}", mat_id=mat, dx=dx, materials=[material], freq=freq,
                ports=[port])


def config2():
    """BASELINE configs[1]: thin-film meander over a ground plane, 256x32x4, dx 0.1 um.

    z=0 full ground; z=1 a 4x4 via at x[2,6) y[26,30); z=2..3 a 4-wide meander
    (SURVEY 8(d) config 2).  Port between the strip start and the ground at x=0.
    """
    Kx, Ky, Kz = 256, 32, 4
    m = np.zeros((Kz, Ky, Kx), dtype=np.uint8)
    _box(m, (0, 0, 0), (Kx, Ky, 1))
    _box(m, (2, 26, 1), (6, 30, 2))
    for lo, hi in [((0, 2), (254, 6)), ((250, 2), (254, 14)), ((2, 10), (254, 14)),
                   ((2, 10), (6, 22)), ((2, 18), (254, 22)), ((250, 18), (254, 30)),
                   ((2, 26), (254, 30))]:
        _box(m, (lo[0], lo[1], 2), (hi[0], hi[1], 4))
    port = {"plus": [(0, -1, (0, 2, 2), (1, 6, 4))], "minus": [(0, -1, (0, 2, 0), (1, 6, 1))]}
    return dict(name="cfg2_meander_256x32x4", mat_id=m, dx=0.1e-6, materials=[NB],
                freqs=list(np.geomspace(1e9, 50e9, 5)), freq=10e9, ports=[port], tucker_tol=1e-6)


def _holes(g, m, z0, z1, n, lo_side, hi_side, keep):
    Kz, Ky, Kx = m.shape
    for _ in range(n):
        s = int(g.integers(lo_side, hi_side + 1))
        x = int(g.integers(0, Kx - s + 1))
        y = int(g.integers(0, Ky - s + 1))
        m[z0:z1, y:y + s, x:x + s] = 0
    for (x0, y0, x1, y1) in keep:
        m[z0:z1, y0:y1, x0:x1] = 1


def config3(seed=3, sigma0=NB[0]):
    """BASELINE configs[2]: 90-degree L strip 8 wide over a holed ground, 512x512x4, dx 0.05 um.

    Two ports, one at each end of the bend (strip against the ground beneath).  An
    8x8 via at the inner corner ties the strip to the ground, so each port sees a
    closed loop and the 2-port Y is non-singular (without a shunt path a series
    element has no Z-parameters; DESIGN.md input recipe).
    """
    Kx, Ky, Kz = 512, 512, 4
    g = rng(seed)
    m = np.zeros((Kz, Ky, Kx), dtype=np.uint8)
    _box(m, (0, 0, 0), (Kx, Ky, 1))
    _holes(g, m, 0, 1, 32, 4, 16, keep=[(0, 256, 8, 264), (256, 504, 264, 512), (256, 256, 264, 264)])
    _box(m, (0, 256, 2), (264, 264, 4))
    _box(m, (256, 256, 2), (264, 512, 4))
    _box(m, (256, 256, 1), (264, 264, 2))   # corner via strip -> ground
    p1 = {"plus": [(0, -1, (0, 256, 2), (1, 264, 4))], "minus": [(0, -1, (0, 256, 0), (1, 264, 1))]}
    p2 = {"plus": [(1, +1, (256, 511, 2), (264, 512, 4))], "minus": [(1, +1, (256, 511, 0), (264, 512, 1))]}
    return dict(name="cfg3_bend_512x512x4", mat_id=m, dx=0.05e-6, materials=[(sigma0, NB[1])],
                freq=10e9, ports=[p1, p2])


def config4(seed=4):
    """BASELINE configs[3]: eSFQ-like 4-metal stack 512x512x16, 16 ports.

    M1 z0-1 holed ground; M2 z4-5 and M4 z12-13 routes along x; M3 z8-9 routes
    along y; each route starts on the domain boundary (its port, against the
    ground face below) and ends in a via stack down to the ground.
    """
    Kx, Ky, Kz = 512, 512, 16
    g = rng(seed)
    m = np.zeros((Kz, Ky, Kx), dtype=np.uint8)
    _box(m, (0, 0, 0), (Kx, Ky, 2))
    routes = []  # (layer z0, axis, lane start, width, length)
    lanes = {4: (0, 6), 12: (6, 11), 8: (11, 16)}
    for zl, (r0, r1) in lanes.items():
        axis = 1 if zl == 8 else 0
        nl = r1 - r0
        for q in range(nl):
            w = int(g.integers(4, 13))
            lane0 = 16 + q * (480 // nl) + int(g.integers(0, (480 // nl) - w))
            length = int(g.integers(160, 480))
            routes.append((zl, axis, lane0, w, length))
    keep, ports, vias = [], [], []
    for zl, axis, l0, w, L in routes:
        if axis == 0:
            _box(m, (0, l0, zl), (L, l0 + w, zl + 2))
            vx = (L - w, l0, L, l0 + w)
            ports.append({"plus": [(0, -1, (0, l0, zl), (1, l0 + w, zl + 2))],
                          "minus": [(0, -1, (0, l0, 0), (1, l0 + w, 2))]})
            keep.append((0, l0, 8, l0 + w))
        else:
            _box(m, (l0, 0, zl), (l0 + w, L, zl + 2))
            vx = (l0, L - w, l0 + w, L)
            ports.append({"plus": [(1, -1, (l0, 0, zl), (l0 + w, 1, zl + 2))],
                          "minus": [(1, -1, (l0, 0, 0), (l0 + w, 1, 2))]})
            keep.append((l0, 0, l0 + w, 8))
        vias.append((vx, zl))
        keep.append(vx)
    _holes(g, m, 0, 2, 64, 4, 16, keep=keep)
    for (x0, y0, x1, y1), zl in vias:
        m[2:zl, y0:y1, x0:x1] = 1
    return dict(name="cfg4_esfq_512x512x16", mat_id=m, dx=0.1e-6, materials=[NB], freq=10e9,
                ports=ports)


def random_fill(shape_xyz, fill=0.5, seed=5, n_mat=1, materials=None, dx=0.1e-6, freq=10e9):
    """BASELINE configs[4]-style Bernoulli-filled grid (x, y, z extents)."""
    g = rng(seed)
    Kx, Ky, Kz = shape_xyz
    occ = g.random((Kz, Ky, Kx)) < fill
    mid = g.integers(1, n_mat + 1, size=(Kz, Ky, Kx))
    m = np.where(occ, mid, 0).astype(np.uint8)
    if not m.any():
        m.flat[0] = 1
    if materials is None:
        materials = [NB] + [(float(g.uniform(1e6, 5e7)), float(g.uniform(40e-9, 400e-9)))
                            for _ in range(n_mat - 1)]
    return dict(name=f"fill{fill}_{Kx}x{Ky}x{Kz}_s{seed}", mat_id=m, dx=dx, materials=materials,
                freq=freq, ports=[])


def layered(shape_xyz, seed=9, n_mat=2, dx=0.1e-6, freq=10e9):
    """Thin-film-like stack with empty rows and empty planes (the structure of configs
    3-4 at test size): a randomly holed plane at z=0, empty z=1, x-running strips at
    z=2 (some rows empty), empty z=3, a few via voxels at z=4, and empty planes above;
    for Kz > 8 the pattern repeats every 8 planes with the top quarter left empty."""
    Kx, Ky, Kz = shape_xyz
    g = rng(seed)
    m = np.zeros((Kz, Ky, Kx), dtype=np.uint8)
    top = Kz - max(1, Kz // 4) if Kz > 2 else Kz
    for z in range(top):
        lz = z % 8
        if lz == 0:
            m[z] = (g.random((Ky, Kx)) < 0.7) * g.integers(1, n_mat + 1, (Ky, Kx))
        elif lz == 2:
            for y in range(0, Ky, 3):
                if g.random() < 0.6:
                    x0 = int(g.integers(0, max(1, Kx // 3)))
                    m[z, y, x0:Kx - int(g.integers(0, max(1, Kx // 3)))] = int(g.integers(1, n_mat + 1))
        elif lz == 4:
            for _ in range(max(1, Kx * Ky // 200)):
                m[z, int(g.integers(0, Ky)), int(g.integers(0, Kx))] = 1
    if not m.any():
        m[0, 0, 0] = 1
    mats = [NB, (5.8e7, float("inf"))][:n_mat]
    return dict(name=f"layered_{Kx}x{Ky}x{Kz}_s{seed}", mat_id=m, dx=dx, materials=mats, freq=freq, ports=[])


def sweep_shapes():
    """BASELINE configs[4] grid list (cubic + slab)."""
    return [(64, 64, 64), (128, 128, 128), (256, 256, 256), (512, 512, 4), (512, 512, 16),
            (512, 512, 64), (1024, 1024, 16), (1024, 1024, 64)]
