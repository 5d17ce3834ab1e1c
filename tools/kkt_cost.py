"""Cost of the default kkt=True against kkt=False on config 4 (device-timed iterations)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2106_15214_b200 as bn
from paper_2106_15214_b200 import synthetic, solver

N = int(sys.argv[1]) if len(sys.argv) > 1 else 4194304
iters = 32
v = synthetic.config4(N=N, dtype=np.float32)
w0, h0 = synthetic.uniform_init(256, N, 12, seed=112)
ctx = solver.get_context(0, "fp32")
ctx.set_dense(v, 0.0)
for kkt in (False, True, False, True):
    ctx.set_factors(w0, h0)
    cfg = bn.SolverConfig(beta=1.5, rank=12, algorithm="jmm", tol=1e-300, kappa=0.0, max_outer_iters=iters)
    ctx.begin(solver.make_params(cfg, 0.0, kkt=kkt), iters)
    ms = ctx.step_timed(iters)
    done, _ = ctx.sync()
    obj, _, kk = ctx.trace(done)
    print(f"kkt={kkt}: {ms / iters:.3f} ms/iteration, launches/iter {ctx.launches_per_iter()}, kkt row {kk[-1]}")
