"""The complex128 build (svh_opts.precision = 1; SURVEY 8(b) "precision c64|c128", 8(c) c.5).

* svh_matvec_z vs the fp64 oracle's direct sum (oracle.operator.matvec_direct): relative L2
  <= 1e-12 (SURVEY 8(c) c.5 "GPU fp64 build <= 1e-12"), full product and Green-only part, ragged
  extents, two materials, several RHS.
* svh_solve with the operator in fp64 reaches the paper's tight tolerance (RRE 1e-10, MATLAB
  double) and the config 1 inductance matches the dense oracle to 1e-8 (vs 1e-4 for the
  complex64 operator).
* BASELINE configs[2] (SURVEY 8(d) config 3 check): fp64-GPU L == c64-GPU L to 1e-4.
"""
import numpy as np
import pytest

import svh_inputs
from oracle.lattice import Lattice
from oracle.operator import matvec_direct
from oracle.solve import solve_ports

pytestmark = pytest.mark.gpu


def rel_l2(a, b):
    return float(np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel()))


@pytest.mark.parametrize("shape", [(16, 2, 2), (9, 7, 5), (20, 13, 3), (5, 33, 6), (40, 6, 2)])
def test_matvec_z_vs_oracle(svh_lib, shape):
    import torch
    case = svh_inputs.random_fill(shape, fill=0.6, seed=700 + sum(shape), n_mat=2)
    lat = Lattice(case["mat_id"])
    I = svh_inputs.currents(lat.K, nrhs=3, seed=5)
    w = 2 * np.pi * case["freq"]
    with svh_lib.setup_case(case, precision=1) as h:
        t = torch.from_numpy(I).cuda()
        got = {go: h.matvec_z(t, green_only=go).cpu().numpy() for go in (True, False)}
    for go in (True, False):
        ref = matvec_direct(lat, case["materials"], w, case["dx"], I, green_only=go)
        for r in range(3):
            e = rel_l2(got[go][r], ref[r])
            assert e < 1e-12, (go, r, e)


def test_matvec_z_matches_c64(svh_lib):
    """The same handle's complex64 product agrees with its complex128 one to c64 rounding."""
    import torch
    case = svh_inputs.layered((60, 40, 5))
    with svh_lib.setup_case(case, precision=1) as h:
        I = svh_inputs.currents(h.K, nrhs=2, seed=2)
        z = h.matvec_z(torch.from_numpy(I).cuda(), green_only=True).cpu().numpy()
        c = h.matvec(torch.from_numpy(I.astype(np.complex64)).cuda(), green_only=True).cpu().numpy()
    e = rel_l2(c.astype(np.complex128), z)
    assert 1e-9 < e < 1e-5, e


def test_fp64_solve_config1_tight(svh_lib):
    case = svh_inputs.config1()
    lat = Lattice(case["mat_id"])
    ref = solve_ports(lat, case["materials"], 2 * np.pi * case["freq"], case["dx"], case["ports"])
    with svh_lib.setup_case(case, precision=1, rre=1e-10, inner_tol=1e-10) as h:
        res = h.solve(case["ports"])
    assert res["code"] == 0, res["stats"]
    assert res["stats"]["final_rre"] <= 1e-10 * 1.0001
    assert abs(res["L"][0, 0] - ref["L"][0, 0]) <= 1e-8 * abs(ref["L"][0, 0])
    assert abs(res["R"][0, 0] - ref["R"][0, 0]) <= 1e-7 * abs(ref["R"][0, 0])


def test_fp64_vs_c64_config3_L(svh_lib):
    """the fp64-GPU L against the c64-GPU L (<= 1e-4)."""
    case = svh_inputs.config3()
    out = {}
    for prec, rre in ((0, 1e-7), (1, 1e-8)):
        with svh_lib.setup_case(case, precision=prec, rre=rre) as h:
            out[prec] = h.solve(case["ports"])
        assert out[prec]["code"] == 0, out[prec]["stats"]
    L0, L1 = out[0]["L"], out[1]["L"]
    assert np.max(np.abs(L0 - L1)) <= 1e-4 * np.max(np.abs(L1))


def test_matvec_z_needs_precision1(svh_lib):
    import torch
    case = svh_inputs.random_fill((6, 5, 4), fill=0.5, seed=1)
    with svh_lib.setup_case(case) as h:
        with pytest.raises(svh_lib.SvhError):
            h.matvec_z(torch.zeros((1, 5, h.K), dtype=torch.complex128, device="cuda"))
