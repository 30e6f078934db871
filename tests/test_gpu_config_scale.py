"""Inductance at configuration scale (VERDICT r1 "What's missing" #5).

* BASELINE configs[1] (256x32x4 meander, K = 16384): the GPU L against golden values written
  by scripts/golden_cfg2.py from the ORACLE ONLY (GMRES on the reduced saddle system with the
  fp64 direct-sum Z and the Eq. 12-15 Schur preconditioner with an exact sparse inverse; that
  solver is pinned to the dense LU oracle in tests/test_oracle_solve.py).  North star: <= 1e-4.
  Also in the paper's storage mode for this config, Tucker tol 1e-6 (BASELINE configs[1]).
* BASELINE configs[2] (512x512x4 bend, 2 ports): invariants the paper fixes -- reciprocity
  Y = Y^T (P12), sigma0 = 0 frequency independence of L (P11, SPEC acceptance #7) and Tucker
  on / off giving the same L (P16; P:247-248 prints the same error 0.0039 for both).
"""
import json
import os

import numpy as np
import pytest

import svh_inputs

pytestmark = pytest.mark.gpu

L_TOL = 1e-4
GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cfg2_L.json")))


@pytest.mark.parametrize("tucker", [0.0, 1e-6])
def test_config2_inductance_vs_oracle_golden(svh_lib, tucker):
    case = svh_inputs.config2()
    assert GOLDEN["K"] == int((case["mat_id"] > 0).sum())
    with svh_lib.setup_case(case, tucker_tol=tucker, rre=1e-7) as h:
        for pt in GOLDEN["points"]:
            h.set_frequency(pt["freq_hz"])
            res = h.solve(case["ports"])
            assert res["code"] == 0, res["stats"]
            L = float(res["L"][0, 0])
            assert abs(L - pt["L_H"]) <= (L_TOL + tucker) * abs(pt["L_H"]), (pt["freq_hz"], L, pt["L_H"])
            assert abs(float(res["R"][0, 0]) - pt["R_ohm"]) <= 1e-3 * abs(pt["R_ohm"])


def _cfg3_L(svh_lib, case, tucker=0.0, freq=None):
    with svh_lib.setup_case(case, tucker_tol=tucker, rre=1e-7) as h:
        if freq is not None:
            h.set_frequency(freq)
        res = h.solve(case["ports"])
    assert res["code"] == 0, res["stats"]
    return res


def test_config3_reciprocity_and_tucker(svh_lib):
    case = svh_inputs.config3()
    dense = _cfg3_L(svh_lib, case)
    Y = dense["Y"]
    assert np.max(np.abs(Y - Y.T)) <= 1e-4 * np.max(np.abs(Y))                   # P12
    assert np.max(np.abs(dense["L"] - dense["L"].T)) <= 1e-4 * np.max(np.abs(dense["L"]))
    assert np.all(np.linalg.eigvalsh(0.5 * (dense["L"] + dense["L"].T)) > 0)
    tuck = _cfg3_L(svh_lib, case, tucker=1e-6)                                  # P16
    assert np.max(np.abs(tuck["L"] - dense["L"])) <= 1e-4 * np.max(np.abs(dense["L"]))


def test_config3_sigma0_zero_frequency_independence(svh_lib):
    case = svh_inputs.config3(sigma0=0.0)
    L1 = _cfg3_L(svh_lib, case, freq=1e9)["L"]
    L10 = _cfg3_L(svh_lib, case, freq=10e9)["L"]
    assert np.max(np.abs(L1 - L10)) <= 1e-4 * np.max(np.abs(L10))                # P11


def test_config2_amg_hierarchy_on_device(svh_lib):
    """H11: the AMG hierarchy is built on the device (double pairwise aggregation, Galerkin
    products, dense coarsest inverse), is deterministic (two setups give the bitwise-same
    solve) and coarsens like AGMG's double pairwise scheme: several levels, operator complexity
    well below 2 (aggregates of <= 4 nodes), and a bounded number of inner iterations per
    preconditioner apply at the paper's inner solver."""
    case = svh_inputs.config2()
    pt = GOLDEN["points"][0]
    res = []
    for _ in range(2):
        with svh_lib.setup_case(case, tucker_tol=0.0, rre=1e-7) as h:
            h.set_frequency(pt["freq_hz"])
            res.append(h.solve(case["ports"]))
    a, b = res
    assert a["code"] == 0 and b["code"] == 0
    st = a["stats"]
    assert st["amg_levels"] >= 3, st
    assert 1.0 < st["amg_op_complexity"] < 2.0, st
    assert st["t_precond_setup_s"] > 0
    assert np.array_equal(a["Y"], b["Y"])                     # deterministic hierarchy and solve
    assert abs(float(a["L"][0, 0]) - pt["L_H"]) <= L_TOL * abs(pt["L_H"])
    # inner PCG iterations per preconditioner apply (one apply per GMRES iteration + 1)
    per_apply = st["inner_iterations"] / max(1, st["total_iterations"] + 1)
    assert per_apply <= 30, st
