"""Time to the port L-matrix with the Table V stage split: setup (lattice, kernels,
spectra), AMG hierarchy + solve (GMRES iterations, inner PCG iterations, matvec and preconditioner
wall time), and the Schur solver's setup time and memory (Table IV: AMG-PCG vs the sparse-direct
comparator, --schur 1).  usage: python scripts/solve_profile.py cfg3 [cfg4 ...] [--inner-tol 1e-3] [--schur 0|1]"""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import svh_inputs  # noqa: E402
from paper_2105_08627_b200 import svh  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workloads", nargs="+")
    ap.add_argument("--inner-tol", type=float, default=1e-3)
    ap.add_argument("--rre", type=float, default=1e-6)
    ap.add_argument("--schur", type=int, default=0, help="0 = AMG-PCG (P:166), 1 = sparse Cholesky (f4)")
    a = ap.parse_args()
    for w in a.workloads:
        case = {"cfg1": svh_inputs.config1, "cfg2": svh_inputs.config2, "cfg3": svh_inputs.config3,
                "cfg4": svh_inputs.config4}[w]()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        h = svh.setup_case(case, tucker_tol=0.0, inner_tol=a.inner_tol, rre=a.rre, schur_solver=a.schur)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        try:
            res = h.solve(case["ports"])
        except svh.SvhError as e:   # e.g. the sparse-direct factor does not fit one GPU (cfg4)
            print(json.dumps({"workload": case["name"], "K": h.K, "M": h.M, "schur_solver": a.schur,
                              "error": str(e)}), flush=True)
            h.close()
            torch.cuda.empty_cache()
            continue
        t2 = time.perf_counter()
        st = res["stats"]
        print(json.dumps({"workload": case["name"], "K": h.K, "M": h.M, "ports": len(case["ports"]),
                          "inner_tol": a.inner_tol, "rre": a.rre, "setup_s": round(t1 - t0, 3),
                          "solve_s": round(t2 - t1, 3), "gmres_iterations": st["total_iterations"],
                          "inner_pcg_iterations": st["inner_iterations"], "t_matvec_s": round(st["t_matvec_s"], 3),
                          "t_precond_s": round(st["t_precond_s"], 3), "converged": st["converged"],
                          "schur_solver": ["amg_pcg", "sparse_cholesky"][a.schur],
                          "t_precond_setup_s": round(st["t_precond_setup_s"], 3),
                          "precond_MB": round(st["precond_bytes"] / 1e6, 1),
                          "amg_levels": st["amg_levels"], "amg_op_complexity": round(st["amg_op_complexity"], 3),
                          "final_rre": st["final_rre"],
                          "L_pH_diag": [round(float(x) * 1e12, 5) for x in res["L"].diagonal()]}), flush=True)
        h.close()


if __name__ == "__main__":
    main()
