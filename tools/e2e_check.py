"""Time one warm fit() on pinned host V (config 4) with the context's per-pass event profiling
off and on -- the bench's device-timed region switches profiling on before its e2e leg."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2106_15214_b200 as bn
from paper_2106_15214_b200 import synthetic, solver
N = 4194304
v = synthetic.config4(N=N, dtype=np.float32)
w0, h0 = synthetic.uniform_init(256, N, 12, seed=112)
vp = torch.from_numpy(v).pin_memory().numpy()
cfg = bn.SolverConfig(beta=1.5, rank=12, algorithm="jmm", tol=1e-300, kappa=0.0, max_outer_iters=50)
ctx = solver.get_context(0, "fp32")
for prof in (False, True, False):
    ctx.set_profiling(prof)
    bn.fit(vp, cfg, init=(w0, h0), dtype="fp32", kkt=False)
    t = time.perf_counter()
    r = bn.fit(vp, cfg, init=(w0, h0), dtype="fp32", kkt=False)
    dt = time.perf_counter() - t
    print(f"profiling={prof}: fit {dt:.3f} s -> {50 / dt:.1f} it/s; loop {r.trace[-1].seconds:.3f} s")
