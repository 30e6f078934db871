"""Dense matvecs on a config-5 grid, per-pass times (perf probe for the z pass; ncu target).
usage: python scripts/zprobe.py KX KY KZ NRHS"""
import sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import svh_inputs  # noqa: E402
from paper_2105_08627_b200 import svh  # noqa: E402

kx, ky, kz, nrhs = (int(a) for a in sys.argv[1:5])
case = svh_inputs.random_fill((kx, ky, kz), fill=0.5, seed=5)
with svh.setup_case(case) as h:
    I = torch.from_numpy(svh_inputs.currents(h.K, nrhs, seed=1).astype(np.complex64)).cuda()
    out = torch.empty_like(I)
    for _ in range(2):
        h.matvec(I, out=out)
    torch.cuda.synchronize()
    h.profile(True)
    h.matvec(I, out=out)
    torch.cuda.synchronize()
    ms, n = h.profile_read(reset=True)
print("embedding", h.embedding, "passes_ms", dict(zip("ABCDE", np.round(ms, 3))))
