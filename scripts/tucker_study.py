"""circulant Tucker rank / compression / overhead scaling (paper Figs. 2-3,
P:204-216) on the paper's workload shapes: a 2-D plate (L x L x 3 voxels, dx = 1 um) and a
3-D cube (L^3), tol 1e-4.  Synthetic full-fill geometries (the paper's exact structures are
not in the container; ranks depend only on the grid extents).

CR_octant = our dense fp32 octant spectra (7 kernels) / Tucker factors+cores;
CR_paper  = the paper's storage model, 7 full complex-double circulant tensors (8 Kt x 16 B
            each) / Tucker bytes ("memory of circulant tensors");
CO        = (Tucker-mode matvec time - dense-mode matvec time) / dense-mode time, i.e. the
            cost of the on-chip restoration relative to one convolution.
Usage: python scripts/tucker_study.py [--tol 1e-4] [--out profiles/r01/tucker_study.md]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import svh_inputs  # noqa: E402
from paper_2105_08627_b200 import svh  # noqa: E402


def time_matvec(h, I, reps=5):
    h.matvec(I)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        h.matvec(I)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def run(shape, tol):
    case = svh_inputs.random_fill(shape, fill=1.0, seed=1, dx=1e-6)
    out = {"grid": list(shape), "Kt": int(np.prod(shape))}
    t0 = time.perf_counter()
    with svh.setup_case(case, tucker_tol=tol) as ht:
        torch.cuda.synchronize()
        out["setup_tucker_s"] = round(time.perf_counter() - t0, 3)
        st = ht.stats()
        nx, ny, nz = ht.embedding
        I = torch.from_numpy(svh_inputs.currents(ht.K, 1, seed=3).astype(np.complex64)).cuda()
        I16 = torch.from_numpy(svh_inputs.currents(ht.K, 16, seed=4).astype(np.complex64)).cuda()
        t_t = time_matvec(ht, I)
        t_t16 = time_matvec(ht, I16, reps=2)
        ranks = st["ranks"]
        out["max_rank"] = max(max(r) for r in ranks)
        out["CR_octant"] = round(st["compression_ratio"], 1)
        dense_oct = 7.0 * (nx // 2 + 1) * (ny // 2 + 1) * (nz // 2 + 1) * 4
        tbytes = dense_oct / st["compression_ratio"]
        out["tucker_MB"] = round(tbytes / 2 ** 20, 3)
        out["CR_paper"] = round(7.0 * nx * ny * nz * 16 / tbytes, 1)
    with svh.setup_case(case, tucker_tol=0.0) as hd:
        t_d = time_matvec(hd, I)
        t_d16 = time_matvec(hd, I16, reps=2)
    out["matvec_dense_ms"] = round(t_d, 3)
    out["matvec_tucker_ms"] = round(t_t, 3)
    out["CO"] = round((t_t - t_d) / t_d, 3)
    out["CO_16rhs"] = round((t_t16 - t_d16) / t_d16, 3)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tol", type=float, default=1e-4)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    rows = []
    for L in (300, 600, 900, 1200, 1400):
        rows.append(dict(kind="plate", **run((L, L, 3), args.tol)))
        print(json.dumps(rows[-1]), flush=True)
    for L in (64, 128, 192, 256):
        rows.append(dict(kind="cube", **run((L, L, L), args.tol)))
        print(json.dumps(rows[-1]), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            f.write(f"# Circulant Tucker scaling (SURVEY 8(f) f3, paper Figs. 2-3), tol {args.tol:g}, B200\n\n")
            f.write("| shape | grid | Kt | max rank | Tucker MB | CR octant | CR paper-model | dense matvec ms | "
                    "Tucker matvec ms | CO (1 RHS) | CO (16 RHS) | setup s |\n|---|---|---|---|---|---|---|---|---|---|---|---|\n")
            for r in rows:
                f.write(f"| {r['kind']} | {'x'.join(map(str, r['grid']))} | {r['Kt']} | {r['max_rank']} | "
                        f"{r['tucker_MB']} | {r['CR_octant']} | {r['CR_paper']} | {r['matvec_dense_ms']} | "
                        f"{r['matvec_tucker_ms']} | {r['CO']} | {r['CO_16rhs']} | {r['setup_tucker_s']} |\n")


if __name__ == "__main__":
    main()
