import cProfile, pstats, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2106_15214_b200 as bn
from paper_2106_15214_b200 import synthetic
N = 4194304
v = synthetic.config4(N=N, dtype=np.float32)
w0, h0 = synthetic.uniform_init(256, N, 12, seed=112)
vp = torch.from_numpy(v).pin_memory().numpy()
cfg = bn.SolverConfig(beta=1.5, rank=12, algorithm="jmm", tol=1e-300, kappa=0.0, max_outer_iters=50)
bn.fit(vp, cfg, init=(w0, h0), dtype="fp32")   # warm
t = time.perf_counter()
pr = cProfile.Profile(); pr.enable()
r = bn.fit(vp, cfg, init=(w0, h0), dtype="fp32")
pr.disable()
print("fit s", time.perf_counter() - t)
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
# raw pinned H2D bandwidth of this box for reference
x = torch.from_numpy(vp)
torch.cuda.synchronize()
t = time.perf_counter()
y = x.to("cuda", non_blocking=True)
torch.cuda.synchronize()
print("torch pinned H2D GB/s", vp.nbytes / (time.perf_counter() - t) / 1e9)
