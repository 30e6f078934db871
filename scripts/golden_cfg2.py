"""Golden inductance of BASELINE configs[1] (256x32x4 meander, K = 16384) from the ORACLE ONLY:
GMRES(50) on the reduced saddle system with the oracle's fp64 direct-sum Z (every voxel pair
integrated, no FFT) and the Eq. 12-15 Schur preconditioner with an exact sparse inverse
(oracle.solve.solve_ports_iterative, pinned to the dense LU oracle in tests/test_oracle_solve.py).
SURVEY 8(c) c.2 step 5.  Writes tests/golden/cfg2_L.json.

usage: python scripts/golden_cfg2.py [--workers 8]"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import svh_inputs  # noqa: E402
from oracle.lattice import Lattice  # noqa: E402
from oracle.solve import solve_ports_iterative  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", type=int, default=os.cpu_count())
    ap.add_argument("--freqs", type=float, nargs="*", default=[1e9, 50e9])
    a = ap.parse_args()
    case = svh_inputs.config2()
    lat = Lattice(case["mat_id"])
    out = {"case": case["name"], "K": int(lat.K), "M": int(lat.M), "dx": case["dx"],
           "materials": case["materials"], "how": __doc__.split("\n\n")[0].replace("\n", " "),
           "rtol": 1e-10, "points": []}
    for f in a.freqs:
        t0 = time.time()
        r = solve_ports_iterative(lat, case["materials"], 2 * np.pi * f, case["dx"], case["ports"], rtol=1e-10,
                                  workers=a.workers)
        pt = {"freq_hz": f, "L_H": float(r["L"][0, 0]), "R_ohm": float(r["R"][0, 0]),
              "Z_re": float(r["Z"][0, 0].real), "Z_im": float(r["Z"][0, 0].imag), "gmres": r["info"],
              "seconds": round(time.time() - t0, 1)}
        out["points"].append(pt)
        print(json.dumps(pt), flush=True)
    json.dump(out, open(os.path.join(ROOT, "tests", "golden", "cfg2_L.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
