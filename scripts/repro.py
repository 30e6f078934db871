import sys, numpy as np, torch
sys.path.insert(0, '.')
import svh_inputs
from paper_2105_08627_b200 import svh
shape = tuple(int(v) for v in sys.argv[1].split('x'))
case = svh_inputs.random_fill(shape, fill=0.5, seed=3 + sum(shape), n_mat=2)
with svh.setup_case(case) as h:
    I = torch.from_numpy(svh_inputs.currents(h.K, 3, seed=1).astype(np.complex64)).cuda()
    for go in (True, False):
        out = h.matvec(I, green_only=go)
        torch.cuda.synchronize()
    print('ok', shape, h.embedding, float(out.abs().max()))
