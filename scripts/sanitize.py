"""Small matvec / Tucker / slab / solve invocations for compute-sanitizer (SURVEY §4:
memcheck / racecheck / synccheck on configs 1-2-sized problems, one tool per run).
Exercises every production pass kernel with tiny launches."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import svh_inputs  # noqa: E402
from paper_2105_08627_b200 import svh  # noqa: E402
from paper_2105_08627_b200.parallel import SlabMatvec  # noqa: E402

for case in (svh_inputs.config1(), svh_inputs.layered((256, 64, 6))):
    with svh.setup_case(case) as h:
        I = torch.from_numpy(svh_inputs.currents(h.K, 2, seed=0).astype(np.complex64)).cuda()
        h.matvec(I)
        g = torch.zeros((1, 5) + h.shape, dtype=torch.complex64, device="cuda")
        h.matvec_grid(g)
        SlabMatvec(h, 2).matvec_virtual(g)
    torch.cuda.synchronize()
with svh.setup_case(svh_inputs.layered((96, 40, 6)), tucker_tol=1e-6) as h:
    I = torch.from_numpy(svh_inputs.currents(h.K, 2, seed=1).astype(np.complex64)).cuda()
    h.matvec(I)
case = svh_inputs.config1()
with svh.setup_case(case) as h:
    res = h.solve(case["ports"])
print("sanitize run done, L =", res["L"])
