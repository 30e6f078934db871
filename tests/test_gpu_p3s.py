"""GPU parity of plan P3s (SURVEY 8(a) "(H4-H8 fused)", 8(d)).

P3s computes the same Eq. 9 product as P5 with the y and z passes fused on chip
per kx slab; it is forced here with opts.plan = 3 and compared element by element with the
fp64 oracle's direct sum (oracle.operator.matvec_direct), full product and Green-only part
(SURVEY 8(c) c.5), packed and grid layouts, dense and Tucker spectra, at every x / y / z
extent the plan accepts (Nx 128..1024, Ny 8..1024, Nz 1..8) with ragged K, empty rows,
empty planes and dead 16/32-row blocks.  The production configs it runs (cfg2 256x32x4,
cfg3 512x512x4) are checked at full size on sampled observers, and P3s == P5 to c64
rounding on them.
"""
import numpy as np
import pytest

import svh_inputs
from oracle.lattice import Lattice
from oracle.operator import matvec_direct

pytestmark = pytest.mark.gpu

TOL = 1e-5   # north_star: complex64 matvec vs the fp64 oracle, relative L2
SAMPLE_ABOVE = 6000


def rel_l2(a, b):
    return float(np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel()))


def _check(svh_lib, case, nrhs, seed, plan=3, tucker_tol=0.0, tol=TOL, rows=None, grid=False):
    import torch
    lat = Lattice(case["mat_id"])
    I = svh_inputs.currents(lat.K, nrhs=nrhs, seed=seed)
    w = 2 * np.pi * case["freq"]
    if rows is None and lat.K > SAMPLE_ABOVE:
        # the oracle's direct sum costs K^2: larger grids are checked on 48 sampled observers
        # (every source), element by element
        rows = np.sort(np.random.default_rng(seed).choice(lat.K, 48, replace=False))
    got = {}
    with svh_lib.setup_case(case, tucker_tol=tucker_tol, plan=plan) as h:
        if grid:
            kz, ky, kx = case["mat_id"].shape
            vox = (lat.coords[:, 2] * ky + lat.coords[:, 1]) * kx + lat.coords[:, 0]   # x-fastest cells
            Ig = np.zeros((nrhs, 5, kz * ky * kx), dtype=np.complex64)
            Ig[:, :, vox] = I
            t = torch.from_numpy(Ig.reshape(nrhs, 5, kz, ky, kx)).cuda()
            for go in (True, False):
                o = h.matvec_grid(t, green_only=go).cpu().numpy().reshape(nrhs, 5, -1)
                empty = np.ones(kz * ky * kx, bool)
                empty[vox] = False
                assert np.all(o[:, :, empty] == 0), "grid output must be zero at empty voxels"
                got[go] = o[:, :, vox].astype(np.complex128)
        else:
            t = torch.from_numpy(I.astype(np.complex64)).cuda()
            for go in (True, False):
                got[go] = h.matvec(t, green_only=go).cpu().numpy().astype(np.complex128)
        used = h.matvec_plan()[0]
    assert used == plan, used
    for go in (True, False):
        ref = matvec_direct(lat, case["materials"], w, case["dx"], I, green_only=go, rows=rows)
        g = got[go] if rows is None else got[go][:, :, rows]
        for r in range(nrhs):
            e = rel_l2(g[r], ref[r])
            assert e < tol, (go, r, e)


# (Kx, Ky, Kz): x extents 128..1024 (Kx = 64..512 plus ragged), y extents 8..1024, z 2..8
SHAPES = [(64, 4, 2), (100, 6, 3), (200, 12, 4), (300, 20, 2), (512, 8, 1), (512, 8, 2), (70, 33, 4),
          (65, 130, 3), (64, 260, 2), (100, 512, 2), (300, 200, 1), (90, 300, 4)]


@pytest.mark.parametrize("shape", SHAPES)
def test_p3s_random_fill(svh_lib, shape):
    case = svh_inputs.random_fill(shape, fill=0.5, seed=300 + sum(shape), n_mat=2)
    _check(svh_lib, case, 2, 11 + shape[0])


@pytest.mark.parametrize("shape", [(100, 40, 4), (300, 70, 3), (64, 200, 4)])
def test_p3s_layered(svh_lib, shape):
    """Stacks with empty rows, empty planes and dead row blocks (pruning paths)."""
    _check(svh_lib, svh_inputs.layered(shape), 2, 5)


@pytest.mark.parametrize("shape", [(100, 40, 4), (70, 33, 3)])
def test_p3s_grid_layout(svh_lib, shape):
    _check(svh_lib, svh_inputs.layered(shape), 1, 8, grid=True)


@pytest.mark.parametrize("shape,tol", [((100, 40, 4), 1e-6), ((200, 100, 3), 1e-4), ((64, 300, 3), 1e-6)])
def test_p3s_tucker(svh_lib, shape, tol):
    case = svh_inputs.random_fill(shape, fill=0.5, seed=400 + sum(shape), n_mat=2)
    _check(svh_lib, case, 2, 3, tucker_tol=tol, tol=tol + TOL)


def test_p3s_many_rhs(svh_lib):
    """RHS loop inside the slab CTA (kernel values reused across RHS)."""
    case = svh_inputs.random_fill((80, 50, 3), fill=0.5, seed=17, n_mat=2)
    _check(svh_lib, case, 7, 21)


def test_p3s_cfg2_full(svh_lib):
    """BASELINE configs[1] (256x32x4 meander, Tucker 1e-6), full product vs the oracle."""
    _check(svh_lib, svh_inputs.config2(), 1, 2, tucker_tol=1e-6, tol=1e-6 + TOL)


def test_p3s_cfg3_sampled(svh_lib):
    """BASELINE configs[2] (512x512x4 bend with its via: 4 non-empty planes, so the kernel values
    come from the kx-major octant copy) at full size: 3 sampled observers."""
    case = svh_inputs.config3()
    lat = Lattice(case["mat_id"])
    rows = np.sort(np.random.default_rng(6).choice(lat.K, 3, replace=False))
    _check(svh_lib, case, 1, 31, rows=rows)


@pytest.mark.parametrize("which", ["cfg3", "fill512x256x4", "fill512x512x4"])
def test_p3s_equals_p5(svh_lib, which):
    """Same product as P5 on full-size grids (c64 rounding), and auto plan selection picks one."""
    import torch
    case = svh_inputs.config3() if which == "cfg3" else \
        svh_inputs.random_fill(tuple(int(v) for v in which[4:].split("x")), fill=0.5, seed=5)
    outs = {}
    for plan in (5, 3, 0):
        with svh_lib.setup_case(case, plan=plan) as h:
            I = torch.from_numpy(svh_inputs.currents(h.K, 2, seed=9).astype(np.complex64)).cuda()
            outs[plan] = h.matvec(I, green_only=True).cpu().numpy().astype(np.complex128)
            if plan == 0:
                p, t5, t3 = h.matvec_plan()
                assert p in (3, 5) and t5 > 0 and t3 > 0
    assert rel_l2(outs[3], outs[5]) < 2e-6
    assert rel_l2(outs[0], outs[5]) < 2e-6


@pytest.mark.parametrize("shape,tucker", [((64, 8, 16), 0.0), ((100, 512, 4), 1e-6)])
def test_p3s_rejects_ineligible(svh_lib, shape, tucker):
    """plan = 3 on a grid P3s does not cover fails loudly at the first matvec: Nz = 32, and a
    Tucker run whose slab + on-chip kernel values exceed shared memory (4 planes x 1024 ky);
    auto selection takes P5 there."""
    import torch
    case = svh_inputs.random_fill(shape, fill=0.5, seed=1)
    with svh_lib.setup_case(case, plan=3, tucker_tol=tucker) as h:
        I = torch.zeros((1, 5, h.K), dtype=torch.complex64, device="cuda")
        with pytest.raises(svh_lib.SvhError):
            h.matvec(I)
    with svh_lib.setup_case(case, plan=0, tucker_tol=tucker) as h:
        I = torch.zeros((1, 5, h.K), dtype=torch.complex64, device="cuda")
        h.matvec(I)
        assert h.matvec_plan()[0] == 5


def test_p3s_shared_memory_attribute_is_not_lowered(svh_lib):
    """One k_p3_yz instantiation (Nx 128, Ny 512, Nz 8) run with 4, then 3, then 4 non-empty
    planes in one process: its slab is 82 KB, 61 KB, 82 KB of dynamic shared memory.  The
    opt-in size attribute is sticky per kernel, so the cached launch set-up must never lower it
    (the third product would fail to launch)."""
    for kz, seed in ((4, 1), (3, 2), (4, 3)):
        case = svh_inputs.random_fill((64, 200, kz), fill=0.5, seed=700 + kz, n_mat=2)
        _check(svh_lib, case, 1, seed)
