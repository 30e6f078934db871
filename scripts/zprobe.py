"""One dense matvec on a config-5 cube (perf probe for the z pass; ncu target)."""
import sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import svh_inputs  # noqa: E402
from paper_2105_08627_b200 import svh  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 8
case = svh_inputs.random_fill((n, n, n), fill=0.5, seed=5)
with svh.setup_case(case) as h:
    I = torch.from_numpy(svh_inputs.currents(h.K, nrhs, seed=1).astype(np.complex64)).cuda()
    out = torch.empty_like(I)
    for _ in range(3):
        h.matvec(I, out=out)
    torch.cuda.synchronize()
print("ok")
