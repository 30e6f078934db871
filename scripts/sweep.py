"""BASELINE configs[4] / SURVEY 8(d) config 5: matvec throughput sweep on 50 % Bernoulli fills
(seed 5), cubic and slab grids, dense octant spectra and Tucker ranks, batches of RHS.
Prints one JSON line per point and writes a markdown table.
Usage: python scripts/sweep.py [--out profiles/r01/sweep_cfg5.md] [--quick]"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import svh_inputs  # noqa: E402
from paper_2105_08627_b200 import svh  # noqa: E402


def bench_point(shape, nrhs, tucker, reps=5):
    case = svh_inputs.random_fill(shape, fill=0.5, seed=5)
    with svh.setup_case(case, tucker_tol=tucker) as h:
        I = torch.from_numpy(svh_inputs.currents(h.K, nrhs, seed=1).astype(np.complex64)).cuda()
        out = torch.empty_like(I)
        h.matvec(I, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            h.matvec(I, out=out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        h.profile(True)
        h.matvec(I, out=out)
        torch.cuda.synchronize()
        pms, pn = h.profile_read(reset=True)
        h.profile(False)
        passes = {n: round(float(x), 3) for n, x in zip("ABCDE", pms[:5])}
        st = h.stats()
        nx, ny, nz = h.embedding
        kt = int(np.prod(shape))
        # P5 bytes (1081 B per voxel per RHS) as the plan-independent yardstick
        p5 = 1081.0 * kt * nrhs
        return {"grid": "x".join(map(str, shape)), "embedding": f"{nx}x{ny}x{nz}", "nrhs": nrhs,
                "kernels": f"tucker {tucker:g} (max rank {max(max(r) for r in st['ranks'])})" if tucker else "dense",
                "ms": round(ms, 3), "Gvu_s": round(5 * kt * nrhs / (ms / 1e3) / 1e9, 2),
                "P5_equiv_TBs": round(p5 / (ms / 1e3) / 1e12, 2), "passes_ms": passes}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--min-kz", type=int, default=0, help="only the points with K_z >= this")
    ap.add_argument("--dense-only", action="store_true")
    args = ap.parse_args()
    pts = [((64, 64, 64), 16, 0.0), ((128, 128, 128), 8, 0.0), ((256, 256, 256), 2, 0.0),
           ((512, 512, 4), 16, 0.0), ((512, 512, 16), 16, 0.0), ((512, 512, 64), 4, 0.0),
           ((1024, 1024, 16), 4, 0.0), ((1024, 1024, 64), 2, 0.0),
           ((512, 512, 16), 1, 0.0), ((512, 512, 16), 4, 0.0), ((512, 512, 16), 64, 0.0),
           ((512, 512, 16), 16, 1e-4), ((512, 512, 16), 16, 1e-8), ((128, 128, 128), 8, 1e-6)]
    pts = [p for p in pts if p[0][2] >= args.min_kz and not (args.dense_only and p[2])]
    rows = []
    for shape, nrhs, tol in pts:
        try:
            r = bench_point(shape, nrhs, tol)
        except Exception as e:   # e.g. out of memory for a large batch
            r = {"grid": "x".join(map(str, shape)), "nrhs": nrhs, "error": str(e)[:120]}
        rows.append(r)
        print(json.dumps(r), flush=True)
        torch.cuda.empty_cache()
    if args.out:
        lines = ["# Matvec throughput sweep (BASELINE configs[4], SURVEY 8(d) config 5), B200, c64, 50% fill\n",
                 "P5-equivalent = 1081 B/voxel/RHS / time (SURVEY 8(d) plan-independent yardstick; 6.44 TB/s = "
                 "100 % of the measured copy bandwidth).\n",
                 "| grid | embedding | RHS | kernels | ms / matvec | G voxel-unknowns/s | P5-equiv TB/s |",
                 "|---|---|---|---|---|---|---|"]
        for r in rows:
            if "error" in r:
                lines.append(f"| {r['grid']} | - | {r['nrhs']} | - | error: {r['error']} | - | - |")
            else:
                lines.append(f"| {r['grid']} | {r['embedding']} | {r['nrhs']} | {r['kernels']} | {r['ms']} | "
                             f"{r['Gvu_s']} | {r['P5_equiv_TBs']} |")
        open(args.out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
