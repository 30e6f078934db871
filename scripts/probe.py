"""Per-pass matvec timing on one grid (perf probe; not a bench line).

usage: python scripts/probe.py SHAPE NRHS [TUCKER_TOL] [--reps N]
  SHAPE = KXxKYxKZ (50 % Bernoulli fill, seed 5) or cfg3 / cfg4
Prints one JSON line: ms per matvec (CUDA events, mean of reps), per-pass ms, the
algorithmic bytes of each pass and its fraction of MEASURED_PEAKS hbm_gbs."""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import svh_inputs  # noqa: E402
from paper_2105_08627_b200 import svh  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("shape")
    ap.add_argument("nrhs", type=int)
    ap.add_argument("tol", type=float, nargs="?", default=0.0)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    if a.shape == "cfg4":
        case = svh_inputs.config4()
    elif a.shape == "cfg3":
        case = svh_inputs.config3()
    else:
        case = svh_inputs.random_fill(tuple(int(v) for v in a.shape.split("x")), fill=0.5, seed=5)
    sys.path.insert(0, ROOT)
    from bench import pass_bytes, load_peaks
    peak = load_peaks()[0]["hbm_gbs"]
    with svh.setup_case(case, tucker_tol=a.tol) as h:
        I = torch.from_numpy(svh_inputs.currents(h.K, a.nrhs, seed=1).astype(np.complex64)).cuda()
        out = torch.empty_like(I)
        for _ in range(2):
            h.matvec(I, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            h.matvec(I, out=out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        h.profile(True)
        h.matvec(I, out=out)
        torch.cuda.synchronize()
        pms, _ = h.profile_read(reset=True)
        h.profile(False)
        pb = pass_bytes(h, a.nrhs)
        st = h.stats()
        kt = int(np.prod(case["mat_id"].shape))
        res = {"grid": a.shape, "nrhs": a.nrhs, "tol": a.tol, "K": h.K, "embedding": list(h.embedding),
               "max_rank": max(max(r) for r in st["ranks"]) if a.tol else 0,
               "ms": round(ms, 3), "Gvu_s": round(5 * kt * a.nrhs / ms / 1e6, 2),
               "passes": {n: {"ms": round(float(t), 3), "GB": round(b / 1e9, 2),
                              "frac": round(b / (float(t) * 1e-3) / 1e9 / peak, 3)}
                          for n, t, b in zip("ABCDE", pms[:5], pb)},
               "step_frac": round(sum(pb) / (ms * 1e-3) / 1e9 / peak, 3)}
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
