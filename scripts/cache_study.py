"""SURVEY 8(f) f1 / paper Table II: Toeplitz kernels of an L^3 cube by direct
quadrature vs restored from the Algorithm-2 install-time Tucker cache.

Writes a markdown table (memory of the original Toeplitz tensors, cache size on disk, setup
time both ways, max relative kernel difference) -- synthetic full cubes, dx = 1 um.
Usage: python scripts/cache_study.py [--nmax 512] [--tol 1e-10] [--out profiles/r01/cache_study.md]
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import svh_inputs  # noqa: E402
from paper_2105_08627_b200 import svh  # noqa: E402


def setup_time(case, **kw):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h = svh.setup_case(case, **kw)
    torch.cuda.synchronize()
    return h, time.perf_counter() - t0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nmax", type=int, default=512)
    ap.add_argument("--tol", type=float, default=1e-10)
    ap.add_argument("--sizes", default="100,200,300,400,500")
    ap.add_argument("--out", default=None)
    ap.add_argument("--cache", default="/tmp/svh_kernels.svxt")
    args = ap.parse_args()
    svh.lib()
    torch.cuda.init()
    t0 = time.perf_counter()
    svh.kernel_cache_build(args.cache, (args.nmax,) * 3, tol=args.tol)
    t_build = time.perf_counter() - t0
    cache_mb = os.path.getsize(args.cache) / 2 ** 20
    rows = []
    for L in [int(v) for v in args.sizes.split(",")]:
        case = svh_inputs.random_fill((L, L, L), fill=1.0, seed=1, dx=1e-6)
        hd, td = setup_time(case)
        hc, tc = setup_time(case, kernel_cache=args.cache)
        err = None
        if L <= 200:
            kd, kc = hd.kernels(), hc.kernels()
            err = max(float(np.linalg.norm(kc[q] - kd[q]) / np.linalg.norm(kd[q])) for q in range(7))
        hd.close()
        hc.close()
        r = dict(L=L, orig_mb=7 * L ** 3 * 8 / 2 ** 20, td=td, tc=tc, err=err)
        rows.append(r)
        print(r, flush=True)
    lines = [f"# Toeplitz kernels: direct quadrature vs Algorithm-2 Tucker cache (SURVEY 8(f) f1, paper Table II), B200\n",
             f"Cache: Nmax = {args.nmax}^3, tol {args.tol:g}, built once in {t_build:.1f} s, {cache_mb:.2f} MB on disk "
             f"(all 7 kernels).  Setup = the whole svh_setup (lattice, kernels, dense octant spectra); only the "
             f"kernel stage differs.\n",
             "| cube L (voxels) | original Toeplitz MB (7 fp64 tensors) | setup, direct quadrature s | "
             "setup, from cache s | speed-up | max rel. kernel diff |", "|---|---|---|---|---|---|"]
    for r in rows:
        e = f"{r['err']:.1e}" if r["err"] is not None else "-"
        lines.append(f"| {r['L']} | {r['orig_mb']:.1f} | {r['td']:.3f} | {r['tc']:.3f} | {r['td'] / r['tc']:.2f} | {e} |")
    text = "\n".join(lines) + "\n"
    print(text)
    if args.out:
        open(args.out, "w").write(text)


if __name__ == "__main__":
    main()
