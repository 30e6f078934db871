"""GPU parity of the slab-decomposed matvec run as P virtual ranks on one
GPU (the all-to-alls become device copies; the kernels, index maps and buffer layouts are
the multi-GPU ones).  Compared with the single-GPU svh_matvec_grid and with the oracle."""
import numpy as np
import pytest

import svh_inputs
from oracle.lattice import Lattice
from oracle.operator import matvec_direct

pytestmark = pytest.mark.gpu

TOL = 1e-5


def _grid_currents(case, lat, I):
    g = np.zeros((I.shape[0], 5) + case["mat_id"].shape, dtype=np.complex64)
    c = lat.coords
    g[:, :, c[:, 2], c[:, 1], c[:, 0]] = I
    return g


# (40, 8, 40): Nz = 128, the TMA-staged z pass (k_ztma2) on kx-slabs (global kx offset)
@pytest.mark.parametrize("shape,P", [((40, 64, 6), 2), ((40, 64, 6), 4), ((24, 16, 5), 4), ((130, 8, 3), 8),
                                     ((40, 8, 40), 2), ((40, 8, 40), 4)])
@pytest.mark.parametrize("green_only", [False, True])
def test_slab_matvec_virtual(svh_lib, shape, P, green_only):
    import torch
    from paper_2105_08627_b200.parallel import SlabMatvec
    case = svh_inputs.layered(shape) if shape[2] >= 6 else svh_inputs.random_fill(shape, fill=0.5, seed=4, n_mat=2)
    lat = Lattice(case["mat_id"])
    I = svh_inputs.currents(lat.K, 2, seed=31)
    g = torch.from_numpy(_grid_currents(case, lat, I)).cuda()
    with svh_lib.setup_case(case) as h:
        whole = h.matvec_grid(g, green_only=green_only).cpu().numpy()
        slab = SlabMatvec(h, P).matvec_virtual(g, green_only=green_only).cpu().numpy()
    occ = case["mat_id"] > 0
    assert np.all(slab[:, :, ~occ] == 0)
    assert np.linalg.norm(slab - whole) <= 1e-6 * np.linalg.norm(whole)
    ref = matvec_direct(lat, case["materials"], 2 * np.pi * case["freq"], case["dx"], I, green_only=green_only)
    c = lat.coords
    got = slab[:, :, c[:, 2], c[:, 1], c[:, 0]].astype(np.complex128)
    for r in range(2):
        assert np.linalg.norm(got[r] - ref[r]) / np.linalg.norm(ref[r]) < TOL


def test_slab_sizes_and_errors(svh_lib):
    case = svh_inputs.random_fill((24, 16, 5), fill=0.5, seed=4)
    with svh_lib.setup_case(case) as h:
        Kyl, Nxl, chunk, per = h.slab_sizes(4)
        nx, ny, nz = h.embedding
        assert (Kyl, Nxl) == (4, nx // 4) and chunk == 5 * 5 * Kyl * Nxl and per == 4 * chunk
        with pytest.raises(RuntimeError):
            h.slab_sizes(3)          # Ky % P != 0
