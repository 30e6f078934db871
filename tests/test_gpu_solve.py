"""GPU parity of the saddle operator (Eq. 7) and of the port solve (GMRES + Schur/AMG
preconditioner) against the fp64 oracle's dense direct solve.

North star: extracted inductances match the oracle to <= 1e-4 relative.
"""
import numpy as np
import pytest

import svh_inputs
from _pins import bar_closed_form
from oracle.lattice import Lattice
from oracle.operator import dense_Z
from oracle.solve import solve_ports

pytestmark = pytest.mark.gpu

L_TOL = 1e-4


def oracle_L(case):
    lat = Lattice(case["mat_id"])
    return solve_ports(lat, case["materials"], 2 * np.pi * case["freq"], case["dx"], case["ports"])


def gpu_solve(svh_lib, case, **opts):
    with svh_lib.setup_case(case, tucker_tol=0.0, **opts) as h:
        return h.solve(case["ports"])


def test_apply_system_matches_oracle(svh_lib):
    """svh_apply_system = [Z A^T; A 0] [I; Phi] (reading G12) vs the oracle's dense blocks."""
    import torch
    case = svh_inputs.random_fill((7, 5, 3), fill=0.6, seed=21, n_mat=2)
    lat = Lattice(case["mat_id"])
    w = 2 * np.pi * case["freq"]
    Z = dense_Z(lat, case["materials"], w, case["dx"])
    A = lat.incidence().toarray()
    g = np.random.default_rng(3)
    x = (g.standard_normal((2, lat.N)) + 1j * g.standard_normal((2, lat.N)))
    n5 = 5 * lat.K
    ref = np.concatenate([x[:, :n5] @ Z.T + x[:, n5:] @ A, x[:, :n5] @ A.T], axis=1)
    with svh_lib.setup_case(case) as h:
        assert (h.K, h.M) == (lat.K, lat.M)
        y = h.apply_system(torch.from_numpy(x.astype(np.complex64)).cuda()).cpu().numpy()
    for r in range(2):
        assert np.linalg.norm(y[r] - ref[r]) / np.linalg.norm(ref[r]) < 1e-5


def test_config1_inductance(svh_lib):
    """BASELINE configs[0]: GPU L and R vs the dense oracle and the closed form (P9)."""
    case = svh_inputs.config1()
    res = gpu_solve(svh_lib, case, rre=1e-7)
    ref = oracle_L(case)
    L_cf, R_cf = bar_closed_form(16, 2, 2, 0.25e-6, 1.7e7, 90e-9, 10e9)
    assert res["code"] == 0, res
    assert abs(res["L"][0, 0] - ref["L"][0, 0]) < L_TOL * abs(ref["L"][0, 0])
    assert abs(res["L"][0, 0] - L_cf) < L_TOL * L_cf
    assert abs(res["R"][0, 0] - R_cf) < 1e-3 * R_cf
    assert res["stats"]["converged"] == 1


@pytest.mark.parametrize("dims", [(12, 3, 3), (8, 4, 4), (16, 1, 1)])
def test_bar_inductance(svh_lib, dims):
    """Non-uniform current bars (PWL and K1/K2 paths active), sigma0 = 0."""
    case = svh_inputs.bar(*dims, dx=0.25e-6, material=(0.0, 90e-9))
    res = gpu_solve(svh_lib, case, rre=1e-7)
    ref = oracle_L(case)
    assert abs(res["L"][0, 0] - ref["L"][0, 0]) < L_TOL * abs(ref["L"][0, 0])


def test_two_port_random_conductor(svh_lib):
    """2 ports on a ragged random conductor with two materials, a floating piece and a hole."""
    rng = np.random.default_rng(5)
    mat = np.zeros((3, 6, 14), np.uint8)
    mat[0, :, :] = 1
    mat[2, 1:5, 2:12] = 2
    mat[1, 2:4, 2:4] = 2     # via between the layers
    mat[0, 2:4, 6:8] = 0     # hole in the ground
    mat[2, 5, 13] = 1        # floating voxel
    ports = [{"plus": [(0, -1, (0, 0, 0), (1, 6, 1))], "minus": [(0, +1, (13, 0, 0), (14, 6, 1))]},
             {"plus": [(0, +1, (11, 1, 2), (12, 5, 3))], "minus": [(0, +1, (13, 0, 0), (14, 6, 1))]}]
    case = dict(mat_id=mat, dx=0.2e-6, materials=[(1.7e7, 90e-9), (0.0, 150e-9)], freq=5e9, ports=ports)
    res = gpu_solve(svh_lib, case, rre=1e-7)
    ref = oracle_L(case)
    assert res["code"] == 0, res
    assert np.max(np.abs(res["L"] - ref["L"])) < L_TOL * np.max(np.abs(ref["L"]))
    assert np.allclose(res["Y"], res["Y"].T, rtol=1e-4, atol=1e-4 * np.abs(res["Y"]).max())
    del rng


def test_preconditioner_reduces_iterations(svh_lib):
    """SPEC acceptance #6: the Schur/AMG preconditioner converges in few iterations."""
    case = svh_inputs.bar(12, 3, 3, dx=0.25e-6, material=(0.0, 90e-9))
    res = gpu_solve(svh_lib, case, rre=1e-7)
    assert res["stats"]["total_iterations"] < 40


def test_three_port_batched_vs_oracle(svh_lib):
    """3 ports (the batched lockstep FGMRES pads to 4 right-hand-side pairs): L vs the oracle's
    dense solve, reciprocity of Y (P12)."""
    mat = np.zeros((3, 8, 16), np.uint8)
    mat[0, :, :] = 1
    mat[2, 1:3, 1:15] = 1
    mat[2, 5:7, 1:15] = 1
    mat[1, 1:3, 14:15] = 1
    mat[1, 5:7, 14:15] = 1
    g = [(0, -1, (0, 0, 0), (1, 8, 1))]
    ports = [{"plus": [(0, -1, (1, 1, 2), (2, 3, 3))], "minus": g},
             {"plus": [(0, -1, (1, 5, 2), (2, 7, 3))], "minus": g},
             {"plus": [(0, +1, (15, 0, 0), (16, 8, 1))], "minus": g}]
    case = dict(mat_id=mat, dx=0.25e-6, materials=[(1.7e7, 90e-9)], freq=10e9, ports=ports)
    res = gpu_solve(svh_lib, case, rre=1e-7)
    ref = oracle_L(case)
    assert res["code"] == 0, res
    assert np.max(np.abs(res["L"] - ref["L"])) < L_TOL * np.max(np.abs(ref["L"]))
    assert np.allclose(res["Y"], res["Y"].T, rtol=1e-4, atol=1e-4 * np.abs(res["Y"]).max())


def test_config2_frequency_sweep(svh_lib):
    """BASELINE configs[1]: 256x32x4 meander, f = 1-50 GHz over 5 points through
    svh_set_frequency (kernels are f-independent, only z^b and the Green prefactor change):
    equals a fresh setup at each frequency; with sigma0 = 0 the inductance is f-independent
    (P11, SPEC acceptance #7)."""
    case = svh_inputs.config2()
    freqs = np.geomspace(1e9, 50e9, 5)
    with svh_lib.setup_case(case, tucker_tol=0.0, rre=1e-7) as h:
        Ls = []
        for f in freqs:
            h.set_frequency(f)
            Ls.append(float(h.solve(case["ports"])["L"][0, 0]))
    with svh_lib.setup_case(dict(case, freq=freqs[-1]), tucker_tol=0.0, rre=1e-7) as h:
        fresh = float(h.solve(case["ports"])["L"][0, 0])
    assert abs(Ls[-1] - fresh) <= 1e-5 * abs(fresh)
    sc = dict(case, materials=[(0.0, m[1]) for m in case["materials"]])
    with svh_lib.setup_case(sc, tucker_tol=0.0, rre=1e-7) as h:
        L0 = []
        for f in (freqs[0], freqs[-1]):
            h.set_frequency(f)
            L0.append(float(h.solve(sc["ports"])["L"][0, 0]))
    assert abs(L0[0] - L0[1]) <= 1e-4 * abs(L0[0]), L0
