"""Pins for oracle/solve.py (CPU only): closed forms P8-P10, invariants P11-P13."""
import numpy as np
import pytest

import svh_inputs
from _pins import MU0, bar_closed_form
from oracle.lattice import Lattice
from oracle.solve import solve_ports


def run(case, materials=None, freq=None):
    lat = Lattice(case["mat_id"])
    f = case["freq"] if freq is None else freq
    return solve_ports(lat, case["materials"] if materials is None else materials, 2 * np.pi * f, case["dx"],
                       case["ports"], return_fields=True)


@pytest.mark.parametrize("lam", [90e-9, 2e-6])
def test_thin_wire_closed_form(lam):
    """P8: n x 1 x 1 wire with end-face ports: L = mu0 b l/A + mu0 dx S_box(n,1,1) exactly."""
    case = svh_inputs.bar(16, 1, 1, dx=0.25e-6, material=(0.0, lam))
    r = run(case)
    L_ref, R_ref = bar_closed_form(16, 1, 1, 0.25e-6, 0.0, lam, case["freq"])
    assert abs(r["L"][0, 0] - L_ref) < 1e-9 * L_ref
    assert abs(r["R"][0, 0]) < 1e-6 * 2 * np.pi * case["freq"] * L_ref


def test_config1_closed_form():
    """P9: config 1 (16x2x2 Nb bar): the uniform current is exact for a 2x2 cross section,
    L = mu0 b l/A + mu0 dx S_box(16,2,2)/16 and R = a l/A (SURVEY: 2.2760813e-12 H, 1.112416e-4 Ohm)."""
    case = svh_inputs.config1()
    r = run(case)
    L_ref, R_ref = bar_closed_form(16, 2, 2, 0.25e-6, 1.7e7, 90e-9, 10e9)
    assert abs(r["L"][0, 0] - L_ref) < 1e-8 * L_ref
    assert abs(r["R"][0, 0] - R_ref) < 1e-8 * R_ref
    assert abs(L_ref - 2.2760813e-12) < 1e-7 * L_ref   # survey's scratch value, 8 digits


def test_dc_resistance():
    """P10: normal conductor (lambda = inf) at f -> 0: R = l/(sigma0 A) exactly."""
    case = svh_inputs.bar(16, 2, 2, dx=0.25e-6, material=(1.7e7, np.inf), freq=1.0)
    r = run(case)
    R_ref = 16 * 0.25e-6 / (1.7e7 * (0.5e-6) ** 2)
    assert abs(r["R"][0, 0] - R_ref) < 1e-9 * R_ref


def test_interior_bar_below_bound():
    """P9: with interior voxels the uniform current is only feasible -> L < bound (energy minimum)."""
    case = svh_inputs.bar(8, 4, 4, dx=0.25e-6, material=(0.0, 90e-9))
    r = run(case)
    L_bound, _ = bar_closed_form(8, 4, 4, 0.25e-6, 0.0, 90e-9, case["freq"])
    assert 0.9 * L_bound < r["L"][0, 0] < L_bound * (1 - 1e-4)


def test_frequency_independence_sigma0_zero():
    """P11: sigma0 = 0 => L independent of f, |R|/(w|L|) tiny."""
    case = svh_inputs.bar(6, 3, 2, dx=0.25e-6, material=(0.0, 90e-9))
    L1 = run(case, freq=1e9)["L"][0, 0]
    r2 = run(case, freq=1e10)
    assert abs(r2["L"][0, 0] - L1) < 1e-10 * L1
    assert abs(r2["R"][0, 0]) < 1e-6 * 2 * np.pi * 1e10 * L1


def two_port_case():
    """12x1x1 bar, ports at both ends, common ground on the -z face of voxel 6."""
    mat = np.ones((1, 1, 12), np.uint8)
    mat = np.concatenate([mat, np.zeros((1, 1, 12), np.uint8)], 0)
    mat[1, 0, 6] = 1   # a stub above voxel 6 so the ground face is interior-free
    ports = [{"plus": [(0, -1, (0, 0, 0), (1, 1, 1))], "minus": [(2, -1, (6, 0, 0), (7, 1, 1))]},
             {"plus": [(0, +1, (11, 0, 0), (12, 1, 1))], "minus": [(2, -1, (6, 0, 0), (7, 1, 1))]}]
    return dict(mat_id=mat, dx=0.25e-6, materials=[(0.0, 90e-9)], freq=10e9, ports=ports)


def test_reciprocity_and_pd():
    """P12: Y = Y^T, L symmetric and SPD for sigma0 = 0."""
    r = run(two_port_case())
    assert np.allclose(r["Y"], r["Y"].T, rtol=1e-10, atol=0)
    assert np.allclose(r["L"], r["L"].T, rtol=1e-9)
    assert np.all(np.linalg.eigvalsh(r["L"]) > 0)


def test_kcl_and_swap():
    """P13: KCL at the solution; swapping + and - terminals leaves L unchanged (SPEC)."""
    case = svh_inputs.bar(5, 2, 1, dx=0.25e-6, material=(1.7e7, 90e-9))
    r = run(case)
    f = r["fields"][0]
    assert np.linalg.norm(f["kcl"]) < 1e-12 * np.linalg.norm(f["I"])
    p = case["ports"][0]
    case2 = dict(case, ports=[{"plus": p["minus"], "minus": p["plus"]}])
    r2 = run(case2)
    assert abs(r2["L"][0, 0] - r["L"][0, 0]) < 1e-10 * abs(r["L"][0, 0])


def test_floating_conductor_grounded():
    """G14: a conductor touching no port does not make the system singular, and a far
    floating block only perturbs L slightly (it is inductively coupled)."""
    mat = np.zeros((1, 3, 8), np.uint8)
    mat[0, 0, :] = 1
    mat[0, 2, 2:5] = 1   # floating block
    port = {"plus": [(0, +1, (7, 0, 0), (8, 1, 1))], "minus": [(0, -1, (0, 0, 0), (1, 1, 1))]}
    case = dict(mat_id=mat, dx=0.25e-6, materials=[(0.0, 90e-9)], freq=10e9, ports=[port])
    r = run(case)
    L_ref, _ = bar_closed_form(8, 1, 1, 0.25e-6, 0.0, 90e-9, 10e9)
    assert abs(r["L"][0, 0] - L_ref) < 0.05 * L_ref


def test_iterative_oracle_equals_dense():
    """solve_ports_iterative (GMRES + Eq. 12-15 Schur preconditioner + direct-sum Z, the oracle
    used for config-2 golden values) reproduces the dense LU oracle (itself pinned by the P8-P13
    closed forms) on a 2-port conductor and a non-uniform bar."""
    import svh_inputs
    from oracle.solve import solve_ports, solve_ports_iterative
    mat = np.zeros((3, 6, 14), np.uint8)
    mat[0, :, :] = 1
    mat[2, 1:5, 2:12] = 2
    mat[1, 2:4, 2:4] = 2
    mat[0, 2:4, 6:8] = 0
    ports = [{"plus": [(0, -1, (0, 0, 0), (1, 6, 1))], "minus": [(0, +1, (13, 0, 0), (14, 6, 1))]},
             {"plus": [(0, +1, (11, 1, 2), (12, 5, 3))], "minus": [(0, +1, (13, 0, 0), (14, 6, 1))]}]
    cases = [dict(mat_id=mat, dx=0.2e-6, materials=[(1.7e7, 90e-9), (0.0, 150e-9)], freq=5e9, ports=ports),
             svh_inputs.bar(12, 3, 3, dx=0.25e-6, material=(0.0, 90e-9))]
    for case in cases:
        lat = Lattice(case["mat_id"])
        w = 2 * np.pi * case["freq"]
        ref = solve_ports(lat, case["materials"], w, case["dx"], case["ports"])
        it = solve_ports_iterative(lat, case["materials"], w, case["dx"], case["ports"], rtol=1e-11)
        assert all(i["code"] == 0 and i["rre"] < 1e-10 for i in it["info"]), it["info"]
        assert np.max(np.abs(it["L"] - ref["L"])) < 1e-8 * np.max(np.abs(ref["L"]))
