timeout 900 python -m pytest tests/test_gpu_tucker.py -q 2>&1 | tail -5
python - <<'PY'
import sys; sys.path.insert(0,'.')
import time, numpy as np, torch, svh_inputs
from paper_2105_08627_b200 import svh
for shape in [(64,64,64),(256,32,4)]:
    case = svh_inputs.random_fill(shape, fill=1.0, seed=2)
    for tol in (1e-4, 1e-6, 1e-8, 1e-10):
        t0=time.time()
        try:
            with svh.setup_case(case, tucker_tol=tol) as h:
                st = h.stats()
            print(shape, tol, "ranks", [max(r) for r in st["ranks"]], "CR %.1f"%st["compression_ratio"], "%.2fs"%(time.time()-t0))
        except Exception as e:
            print(shape, tol, "ERR", e)
PY
