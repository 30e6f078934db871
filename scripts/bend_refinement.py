"""SURVEY 8(f) f3, refinement consistency on the 90-degree bend (§III.C):
a 2 x 2 mm square-section bend with 10 mm arms, sharp inner edge and outer corner,
lambda_L = 0.45 mm, sigma_0 = 0, discretised with dx = 0.5 ... 0.05 (0.025) mm; the port drives
the end face of one arm against the end face of the other (reading G13).  The paper validates
its dx = 0.025 mm reference by the relative difference to dx = 0.05 mm (8.4e-4) and reports the
relative difference of each coarser dx to the reference (Table III: 0.0039 at dx = 0.1 mm, with
and without Tucker).  This script computes L at every dx on the GPU (svh_setup + svh_solve,
dense and Tucker 1e-8 at dx = 0.1 mm), the relative differences to the finest dx, the
successive-level differences, and the time to L per level.

usage: python scripts/bend_refinement.py [--finest 0.05] [--out profiles/r02/bend_refinement_f3.md]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def bend_case(dx_mm, lam=0.45e-3, arm_mm=10.0, side_mm=2.0, freq=1e9):
    n = int(round(arm_mm / dx_mm))
    w = int(round(side_mm / dx_mm))
    mat = np.zeros((w, n, n), np.uint8)          # [z][y][x]
    mat[:, :w, :] = 1                            # arm A along x (y < w)
    mat[:, :, n - w:] = 1                        # arm B along y (x >= n - w)
    # port: + = -x faces of arm A at x = 0; - = +y faces of arm B at y = n - 1 (ground)
    ports = [{"plus": [(0, -1, (0, 0, 0), (1, w, w))], "minus": [(1, +1, (n - w, n - 1, 0), (n, n, w))]}]
    return dict(name=f"bend_dx{dx_mm}mm", mat_id=mat, dx=dx_mm * 1e-3, materials=[(0.0, lam)], freq=freq,
                ports=ports)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--levels", default="0.5,0.4,0.25,0.2,0.1,0.05")
    ap.add_argument("--tucker-at", type=float, default=0.1)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import torch
    from paper_2105_08627_b200 import svh
    rows = []
    for dx in [float(v) for v in a.levels.split(",")]:
        for tol in ([0.0, 1e-8] if abs(dx - a.tucker_at) < 1e-12 else [0.0]):
            case = bend_case(dx)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            with svh.setup_case(case, tucker_tol=tol, rre=1e-7, inner_tol=1e-3) as h:
                t1 = time.perf_counter()
                res = h.solve(case["ports"])
                t2 = time.perf_counter()
                K, emb = h.K, h.embedding
            st = res["stats"]
            rows.append(dict(dx_mm=dx, tucker=tol, K=K, embedding=list(emb), L_H=float(res["L"][0, 0]),
                             code=res["code"], gmres=st["total_iterations"], inner=st["inner_iterations"],
                             setup_s=round(t1 - t0, 3), solve_s=round(t2 - t1, 3)))
            print(json.dumps(rows[-1]), flush=True)
    dense = [r for r in rows if r["tucker"] == 0.0]
    ref = min(dense, key=lambda r: r["dx_mm"])
    lines = ["# f3: refinement consistency on the 90-degree bend (PAPER.md §III.C, P:234)", "",
             "2 x 2 mm section, 10 mm arms, lambda_L = 0.45 mm, sigma_0 = 0, one port (arm end faces), "
             "B200, `scripts/bend_refinement.py`.  Reference = the finest dx (%g mm)." % ref["dx_mm"], "",
             "| dx (mm) | kernels | K | embedding | L (nH) | rel. diff. to reference | rel. diff. to next finer | "
             "GMRES its | setup s | solve s |", "|---|---|---|---|---|---|---|---|---|---|"]
    for i, r in enumerate(rows):
        finer = [q for q in dense if q["dx_mm"] < r["dx_mm"]]
        nxt = max(finer, key=lambda q: q["dx_mm"]) if finer else None
        d_ref = abs(r["L_H"] - ref["L_H"]) / abs(ref["L_H"])
        d_nxt = abs(r["L_H"] - nxt["L_H"]) / abs(nxt["L_H"]) if nxt else float("nan")
        lines.append("| %g | %s | %d | %s | %.6f | %.3e | %.3e | %d | %.2f | %.2f |" % (
            r["dx_mm"], "Tucker %g" % r["tucker"] if r["tucker"] else "dense", r["K"], "x".join(map(str, r["embedding"])),
            r["L_H"] * 1e9, d_ref, d_nxt, r["gmres"], r["setup_s"], r["solve_s"]))
    lines += ["", "Paper: 8.4e-4 between dx = 0.025 and 0.05 mm; 0.0039 at dx = 0.1 mm against the 0.025 mm "
              "reference, identical with and without Tucker (Table III)."]
    txt = "\n".join(lines) + "\n"
    print(txt)
    if a.out:
        os.makedirs(os.path.dirname(a.out), exist_ok=True)
        open(a.out, "w").write(txt)


if __name__ == "__main__":
    main()
