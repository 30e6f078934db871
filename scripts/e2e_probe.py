import sys, time
sys.path.insert(0, ".")
import numpy as np, torch, svh_inputs
from paper_2105_08627_b200 import svh
case = svh_inputs.config4()
h = svh.setup_case(case)
R = 16
I_host = torch.from_numpy(svh_inputs.currents(h.K, R, seed=1).astype(np.complex64)).pin_memory()
out_host = torch.empty_like(I_host).pin_memory()
I = I_host.cuda(); out = torch.empty_like(I)
for _ in range(3): h.matvec(I, out=out)
torch.cuda.synchronize()
mode = sys.argv[1] if len(sys.argv) > 1 else "a"
if mode == "b":
    h.profile(True); h.profile_read(reset=True)
    for _ in range(20): h.matvec(I, out=out)
    torch.cuda.synchronize()
    h.profile_read(reset=True); h.profile(False)
stream = torch.cuda.current_stream()
h.matvec_host(I_host, out_host); torch.cuda.synchronize()
f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t = time.perf_counter()
f0.record(stream)
for _ in range(20): h.matvec_host(I_host, out_host)
f1.record(stream); torch.cuda.synchronize()
print(mode, "events ms", f0.elapsed_time(f1) / 20, "wall ms", (time.perf_counter() - t) / 20 * 1e3)
