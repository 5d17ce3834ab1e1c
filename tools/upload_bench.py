"""Time Context.set_dense of config-4 V from pinned host memory (5 repeats)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2106_15214_b200 import solver, synthetic
v = synthetic.config4(N=4194304, dtype=np.float32)
vp = torch.from_numpy(v).pin_memory().numpy()
ctx = solver.get_context(0, "fp32")
ts = []
for _ in range(5):
    t = time.perf_counter(); ctx.set_dense(vp, 0.0); ts.append(time.perf_counter() - t)
print("set_dense s", [round(x, 4) for x in ts], "GB/s", round(vp.nbytes / min(ts) / 1e9, 1))
