"""k_zpass (pass C, Nz = 64..256) under compute-sanitizer: small grids that run the dense
(two T buffers) and Tucker (one T buffer, two barriers per tile) variants, the unpredicated
fast path (Kz = N/2, every plane non-empty) and the predicated one (Kz < N/2, empty planes).
Run twice per case and compared bitwise (a race on T or KV would show as run-to-run differences).
usage: [compute-sanitizer --tool racecheck] python scripts/sanitize_zpass.py
(compute-sanitizer is closed on this GPU pool: `profiles/r02/sanitize_zpass_plain_r02h.log` is the plain run.)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import svh_inputs  # noqa: E402
from paper_2105_08627_b200 import svh  # noqa: E402

for shape, tol in (((16, 6, 64), 0.0), ((16, 6, 64), 1e-6), ((16, 5, 40), 1e-6), ((16, 4, 32), 1e-6)):
    case = svh_inputs.random_fill(shape, fill=0.5, seed=5)
    with svh.setup_case(case, tucker_tol=tol) as h:
        I = torch.from_numpy(svh_inputs.currents(h.K, 3, seed=1).astype(np.complex64)).cuda()
        a = h.matvec(I, green_only=True)
        b = h.matvec(I, green_only=True)
        torch.cuda.synchronize()
        assert torch.equal(a, b), "pass C must be deterministic"
        print("zpass sanitize:", shape, "tucker" if tol else "dense", "embedding", h.embedding, "ok", flush=True)
print("sanitize_zpass done")
