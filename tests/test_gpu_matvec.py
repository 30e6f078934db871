"""GPU parity: svh_matvec (CUDA, complex64) vs the fp64 oracle (north star: rel L2 <= 1e-5).

All calls go through the C-ABI (paper_2105_08627_b200.svh).  Both the full
product Z.I and the Green-only part are compared, since the local term can
dominate and would hide FFT errors.
"""
import numpy as np
import pytest

import svh_inputs
from oracle import kernels as okern
from oracle.lattice import Lattice
from oracle.operator import matvec_direct

pytestmark = pytest.mark.gpu

TOL = 1e-5   # BASELINE.json north_star: complex64 matvec vs fp64 oracle, relative L2


def rel_l2(a, b):
    return float(np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel()))


def gpu_matvec(svh_lib, case, I, green_only=False, grid=False, tucker_tol=0.0):
    import torch
    with svh_lib.setup_case(case, tucker_tol=tucker_tol) as h:
        if not grid:
            t = torch.from_numpy(I.astype(np.complex64)).cuda()
            out = h.matvec(t, green_only=green_only)
            torch.cuda.synchronize()
            return out.cpu().numpy().astype(np.complex128)
        lat = Lattice(case["mat_id"])
        g = np.zeros((I.shape[0], 5) + h.shape, dtype=np.complex64)
        c = lat.coords
        g[:, :, c[:, 2], c[:, 1], c[:, 0]] = I
        out = h.matvec_grid(torch.from_numpy(g).cuda(), green_only=green_only).cpu().numpy()
        return out[:, :, c[:, 2], c[:, 1], c[:, 0]].astype(np.complex128)


SMALL = [((1, 1, 1), 1.0), ((2, 1, 1), 1.0), ((16, 2, 2), 1.0), ((5, 3, 2), 0.7), ((13, 7, 3), 0.6),
         ((24, 20, 6), 0.5), ((9, 33, 5), 0.5), ((3, 1, 17), 0.8), ((70, 6, 2), 0.5)]


@pytest.mark.parametrize("shape,fill", SMALL)
def test_kernels_vs_oracle(svh_lib, shape, fill):
    """H2: GPU fp64 quadrature of the 7 kernels vs the oracle at every offset of the grid."""
    case = svh_inputs.random_fill(shape, fill=fill, seed=sum(shape))
    with svh_lib.setup_case(case) as h:
        kg = h.kernels()                       # [7][kz][ky][kx]
    kx, ky, kz = shape
    offs = np.array([(x, y, z) for z in range(kz) for y in range(ky) for x in range(kx)])
    if len(offs) > 400:
        offs = offs[np.random.default_rng(0).choice(len(offs), 400, replace=False)]
    ko = okern.seven_kernels(offs)             # [P][7]
    got = kg[:, offs[:, 2], offs[:, 1], offs[:, 0]].T
    scale = np.abs(ko[:, :1])                  # |K0(m)|
    assert np.max(np.abs(got - ko) / scale) < 1e-11


@pytest.mark.parametrize("shape,fill", SMALL)
@pytest.mark.parametrize("green_only", [False, True])
def test_matvec_small(svh_lib, shape, fill, green_only):
    case = svh_inputs.random_fill(shape, fill=fill, seed=3 + sum(shape), n_mat=2)
    lat = Lattice(case["mat_id"])
    I = svh_inputs.currents(lat.K, nrhs=3, seed=1)
    w = 2 * np.pi * case["freq"]
    ref = matvec_direct(lat, case["materials"], w, case["dx"], I, green_only=green_only)
    got = gpu_matvec(svh_lib, case, I, green_only=green_only)
    for r in range(3):
        assert rel_l2(got[r], ref[r]) < TOL, (r, rel_l2(got[r], ref[r]))


@pytest.mark.parametrize("shape", [(13, 7, 3), (24, 20, 6)])
def test_matvec_grid_layout(svh_lib, shape):
    case = svh_inputs.random_fill(shape, fill=0.5, seed=8, n_mat=2)
    lat = Lattice(case["mat_id"])
    I = svh_inputs.currents(lat.K, nrhs=2, seed=2)
    w = 2 * np.pi * case["freq"]
    ref = matvec_direct(lat, case["materials"], w, case["dx"], I)
    got = gpu_matvec(svh_lib, case, I, grid=True)
    assert rel_l2(got, ref) < TOL


def test_matvec_config1(svh_lib):
    """BASELINE configs[0]: 16x2x2 bar, seeds 0-3."""
    case = svh_inputs.config1()
    lat = Lattice(case["mat_id"])
    w = 2 * np.pi * case["freq"]
    for seed in range(4):
        I = svh_inputs.currents(lat.K, 1, seed=seed)
        for go in (False, True):
            ref = matvec_direct(lat, case["materials"], w, case["dx"], I, green_only=go)
            got = gpu_matvec(svh_lib, case, I, green_only=go)
            assert rel_l2(got, ref) < TOL


def test_matvec_config2_sampled_rows(svh_lib):
    """BASELINE configs[1] at full size (256x32x4 meander): 48 sampled voxels, all 5 components."""
    import torch
    case = svh_inputs.config2()
    lat = Lattice(case["mat_id"])
    rows = np.sort(np.random.default_rng(7).choice(lat.K, 48, replace=False))
    I = svh_inputs.currents(lat.K, 1, seed=11)
    w = 2 * np.pi * case["freq"]
    for go in (True, False):
        ref = matvec_direct(lat, case["materials"], w, case["dx"], I, green_only=go, rows=rows)
        got = gpu_matvec(svh_lib, case, I, green_only=go)[:, :, rows]
        assert rel_l2(got, ref) < TOL


def test_matvec_symmetry_large(svh_lib):
    """Property at any size: Z is complex symmetric (P4/P12), u^T (Z v) = v^T (Z u)."""
    import torch
    case = svh_inputs.random_fill((128, 96, 8), fill=0.5, seed=5)
    with svh_lib.setup_case(case) as h:
        u = torch.from_numpy(svh_inputs.currents(h.K, 1, seed=1).astype(np.complex64)).cuda()
        v = torch.from_numpy(svh_inputs.currents(h.K, 1, seed=2).astype(np.complex64)).cuda()
        for go in (True, False):
            Zv = h.matvec(v, green_only=go).cpu().numpy().astype(np.complex128)
            Zu = h.matvec(u, green_only=go).cpu().numpy().astype(np.complex128)
            a = np.sum(u.cpu().numpy() * Zv)
            b = np.sum(v.cpu().numpy() * Zu)
            assert abs(a - b) / abs(a) < 1e-5


def test_matvec_batch_consistency(svh_lib):
    """nrhs batching (and RHS chunking) gives the same result as single-RHS calls."""
    import torch
    case = svh_inputs.random_fill((40, 12, 5), fill=0.5, seed=12)
    with svh_lib.setup_case(case, rhs_chunk=2) as h:
        I = torch.from_numpy(svh_inputs.currents(h.K, 5, seed=4).astype(np.complex64)).cuda()
        all_ = h.matvec(I).cpu().numpy()
        one = np.stack([h.matvec(I[r]).cpu().numpy() for r in range(5)])
    assert np.array_equal(all_, one)


def test_launch_count_increments(svh_lib):
    import torch
    case = svh_inputs.random_fill((8, 8, 4), fill=0.5, seed=1)
    with svh_lib.setup_case(case) as h:
        I = torch.from_numpy(svh_inputs.currents(h.K, 1, seed=4).astype(np.complex64)).cuda()
        n0 = svh_lib.launch_count()
        h.matvec(I)
        torch.cuda.synchronize()
        assert svh_lib.launch_count() - n0 == 5


# Geometries with empty (y, z) rows and empty z planes: the passes skip them (DESIGN.md
# §5 "pruning"), so these cover every pass path with skipped data -- row passes with
# R2 = 1 and R2 > 1 (Nx = 128 / 256), the strided passes incl. the pipelined inverse
# (Ny = 256), and the z pass with Nz <= 64 and Nz = 256 (k_freq_big).
LAYERED = [(40, 70, 6), (3, 4, 70), (130, 9, 3)]


@pytest.mark.parametrize("shape", LAYERED)
@pytest.mark.parametrize("grid", [False, True])
def test_matvec_pruned_layers(svh_lib, shape, grid):
    case = svh_inputs.layered(shape)
    lat = Lattice(case["mat_id"])
    I = svh_inputs.currents(lat.K, nrhs=2, seed=21)
    w = 2 * np.pi * case["freq"]
    for go in (True, False):
        ref = matvec_direct(lat, case["materials"], w, case["dx"], I, green_only=go)
        got = gpu_matvec(svh_lib, case, I, green_only=go, grid=grid)
        for r in range(2):
            assert rel_l2(got[r], ref[r]) < TOL, (go, r, rel_l2(got[r], ref[r]))


def test_matvec_grid_zero_outside(svh_lib):
    """Grid layout: the output is exactly zero at empty voxels (incl. whole empty rows/planes)."""
    import torch
    case = svh_inputs.layered((40, 70, 6))
    occ = case["mat_id"] > 0
    with svh_lib.setup_case(case) as h:
        assert h.rows_nonempty == int(occ.any(axis=2).sum())
        assert h.planes_nonempty == int(occ.any(axis=(1, 2)).sum())
        g = np.zeros((1, 5) + h.shape, dtype=np.complex64)
        g[:, :, occ] = svh_inputs.currents(int(occ.sum()), 1, seed=3)[0].astype(np.complex64)
        out = h.matvec_grid(torch.from_numpy(g).cuda()).cpu().numpy()
    assert np.all(out[:, :, ~occ] == 0)
    assert np.all(np.isfinite(out))


def test_matvec_host_pipeline(svh_lib):
    """svh_matvec_host (host buffers, chunked H2D / passes / D2H pipeline) equals svh_matvec
    bit for bit, for chunk counts that leave a ragged last chunk."""
    import torch
    case = svh_inputs.layered((40, 70, 6))
    with svh_lib.setup_case(case) as h:
        I = torch.from_numpy(svh_inputs.currents(h.K, 7, seed=9).astype(np.complex64))
        dev = h.matvec(I.cuda()).cpu()
        for chunk in (0, 1, 3, 7):
            out = torch.empty_like(I).pin_memory()
            h.matvec_host(I.pin_memory(), out, chunk=chunk)
            assert torch.equal(out, dev), chunk


# Maximum extents (svh_setup accepts K_i <= 2048 -> embeddings up to 4096 per axis): the
# 4096-point row passes, the 4096-point strided fallback passes and the generic z pass
# (k_freq_big) -- compared with the oracle on sampled output voxels.
MAXES = [(2048, 3, 2), (2, 2048, 2), (3, 2, 1100)]


@pytest.mark.parametrize("shape", MAXES)
def test_matvec_max_extents_sampled(svh_lib, shape):
    case = svh_inputs.random_fill(shape, fill=0.5, seed=sum(shape), n_mat=2)
    lat = Lattice(case["mat_id"])
    rows = np.sort(np.random.default_rng(5).choice(lat.K, 24, replace=False))
    I = svh_inputs.currents(lat.K, 1, seed=17)
    w = 2 * np.pi * case["freq"]
    for go in (True, False):
        ref = matvec_direct(lat, case["materials"], w, case["dx"], I, green_only=go, rows=rows)
        got = gpu_matvec(svh_lib, case, I, green_only=go)[:, :, rows]
        assert rel_l2(got, ref) < TOL, (go, rel_l2(got, ref))


def test_setup_rejects_bad_grids(svh_lib):
    """Degenerate / out-of-range inputs fail loudly through the C-ABI (no silent fallback)."""
    ok = svh_inputs.random_fill((4, 4, 2), fill=0.5, seed=1)
    empty = dict(ok, mat_id=np.zeros_like(ok["mat_id"]))
    with pytest.raises(svh_lib.SvhError):
        svh_lib.setup_case(empty)
    big = dict(ok, mat_id=np.ones((1, 1, 2049), dtype=np.uint8))
    with pytest.raises(svh_lib.SvhError):
        svh_lib.setup_case(big)


# Pass C for 128 <= Nz <= 512 (k_ztma, TMA-staged z pass): Kz = 33..64 -> Nz = 128,
# Kz = 65..128 -> 256, Kz = 129..256 -> 512, incl. Kz = N/2 exactly, a ragged kx tile edge
# in the embedding and 3 RHS (the tile order is RHS-fastest); plus empty planes.
ZSHAPES = [((9, 5, 40), 0.5), ((20, 3, 64), 0.5), ((5, 3, 128), 0.6), ((6, 4, 150), 0.5),
           ((12, 7, 12), 0.5), ((10, 6, 24), 0.5)]   # Nz = 32 / 64 (k_ztma2 opt-in there)


@pytest.mark.parametrize("shape,fill", ZSHAPES)
def test_matvec_ztma_shapes(svh_lib, shape, fill):
    case = svh_inputs.random_fill(shape, fill=fill, seed=31 + sum(shape), n_mat=2)
    lat = Lattice(case["mat_id"])
    I = svh_inputs.currents(lat.K, nrhs=3, seed=5)
    w = 2 * np.pi * case["freq"]
    for go in (True, False):
        ref = matvec_direct(lat, case["materials"], w, case["dx"], I, green_only=go)
        got = gpu_matvec(svh_lib, case, I, green_only=go)
        for r in range(3):
            assert rel_l2(got[r], ref[r]) < TOL, (go, r, rel_l2(got[r], ref[r]))


def test_matvec_ztma_empty_planes(svh_lib):
    """k_ztma over a stack with empty z planes (read as zero, never read back)."""
    case = svh_inputs.layered((8, 6, 100))
    lat = Lattice(case["mat_id"])
    I = svh_inputs.currents(lat.K, nrhs=2, seed=23)
    w = 2 * np.pi * case["freq"]
    ref = matvec_direct(lat, case["materials"], w, case["dx"], I, green_only=True)
    got = gpu_matvec(svh_lib, case, I, green_only=True)
    for r in range(2):
        assert rel_l2(got[r], ref[r]) < TOL, (r, rel_l2(got[r], ref[r]))


# 2048-point y axis (K_y = 513..1024): the TMA-ring strided passes k_ytma<2048> (twiddles from
# the table instead of registers)
@pytest.mark.parametrize("shape", [(3, 600, 2), (2, 1000, 2)])
def test_matvec_y2048(svh_lib, shape):
    case = svh_inputs.random_fill(shape, fill=0.5, seed=41 + sum(shape), n_mat=2)
    lat = Lattice(case["mat_id"])
    I = svh_inputs.currents(lat.K, nrhs=2, seed=8)
    w = 2 * np.pi * case["freq"]
    for go in (True, False):
        ref = matvec_direct(lat, case["materials"], w, case["dx"], I, green_only=go)
        got = gpu_matvec(svh_lib, case, I, green_only=go)
        for r in range(2):
            assert rel_l2(got[r], ref[r]) < TOL, (go, r, rel_l2(got[r], ref[r]))
