"""Time-to-L demo: setup + svh_solve on a BASELINE config; prints L, stats and timings."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import svh_inputs  # noqa: E402
from paper_2105_08627_b200 import svh  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
opts = dict(a.split("=") for a in sys.argv[2:])
case = {"cfg1": svh_inputs.config1, "cfg2": svh_inputs.config2, "cfg3": svh_inputs.config3,
        "cfg4": svh_inputs.config4}[name]()
tol = float(opts.pop("tucker", 0.0))
kw = {k: (float(v) if "." in v or "e" in v else int(v)) for k, v in opts.items()}
torch.cuda.synchronize()
t0 = time.perf_counter()
with svh.setup_case(case, tucker_tol=tol, **kw) as h:
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    res = h.solve(case["ports"])
    t2 = time.perf_counter()
    print(json.dumps({"case": name, "K": h.K, "M": h.M, "N": h.N, "setup_s": t1 - t0, "solve_s": t2 - t1,
                      "L_pH": (res["L"] * 1e12).round(6).tolist(), "R": res["R"].tolist(), "code": res["code"],
                      "stats": res["stats"]}))
