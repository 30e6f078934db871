"""Sparse-direct Schur comparator (the paper's Table IV).

opts.schur_solver = 1 replaces the AMG-preconditioned CG for S^-1 inside the Schur-complement
preconditioner (Eq. 13-15) by a METIS-reordered sparse Cholesky factored once per port set.
The preconditioner changes, the operator and the GMRES target do not, so L must agree with the
oracle (dense LU, config 1 closed form) and with the AMG run to the inductance tolerance; the
direct solve is exact, so the outer FGMRES needs no more iterations than with the inexact AMG
inner solve.  Table IV's trade-off (memory, setup, per-apply time) is reported in the stats.
"""
import json
import os

import numpy as np
import pytest

import svh_inputs
from _pins import bar_closed_form
from oracle.lattice import Lattice
from oracle.solve import solve_ports

pytestmark = pytest.mark.gpu

L_TOL = 1e-4
GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cfg2_L.json")))


def test_direct_config1_closed_form(svh_lib):
    case = svh_inputs.config1()
    with svh_lib.setup_case(case, rre=1e-7, schur_solver=1) as h:
        res = h.solve(case["ports"])
    L_cf, _ = bar_closed_form(16, 2, 2, 0.25e-6, 1.7e7, 90e-9, 10e9)
    assert res["code"] == 0, res
    assert abs(res["L"][0, 0] - L_cf) < L_TOL * L_cf
    st = res["stats"]
    assert st["schur_solver"] == 1 and st["precond_bytes"] > 0


def test_direct_multiport_vs_oracle(svh_lib):
    """3 ports solved in one lockstep batch (the [n][2B] vector layout, B padded to 4): L vs the
    oracle's dense solve (same structure as test_gpu_solve's batched 3-port case)."""
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
    lat = Lattice(case["mat_id"])
    ref = solve_ports(lat, case["materials"], 2 * np.pi * case["freq"], case["dx"], case["ports"])
    with svh_lib.setup_case(case, rre=1e-7, schur_solver=1) as h:
        res = h.solve(case["ports"])
    assert res["code"] == 0
    assert np.max(np.abs(res["L"] - ref["L"])) <= L_TOL * np.max(np.abs(ref["L"]))


def test_direct_config2_golden(svh_lib):
    case = svh_inputs.config2()
    pt = GOLDEN["points"][-1]
    with svh_lib.setup_case(case, rre=1e-7, schur_solver=1) as h:
        h.set_frequency(pt["freq_hz"])
        res = h.solve(case["ports"])
    assert res["code"] == 0, res["stats"]
    assert abs(float(res["L"][0, 0]) - pt["L_H"]) <= L_TOL * abs(pt["L_H"])


def test_direct_vs_amg_config3(svh_lib):
    """BASELINE configs[2] (2 ports): the two Schur solvers give the same L; the exact inner
    solve needs no more outer iterations than the AMG-PCG one."""
    case = svh_inputs.config3()
    out = {}
    for ss in (0, 1):
        with svh_lib.setup_case(case, rre=1e-7, schur_solver=ss, inner_tol=1e-8) as h:
            out[ss] = h.solve(case["ports"])
        assert out[ss]["code"] == 0, out[ss]["stats"]
    La, Ld = out[0]["L"], out[1]["L"]
    assert np.max(np.abs(La - Ld)) <= L_TOL * np.max(np.abs(La))
    assert out[1]["stats"]["total_iterations"] <= out[0]["stats"]["total_iterations"] + 2
    assert out[1]["stats"]["t_precond_setup_s"] > 0 and out[0]["stats"]["t_precond_setup_s"] > 0
