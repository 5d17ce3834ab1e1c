"""Run a few fused iterations on a config-4 column prefix (for ncu captures)."""
import sys, os, time
sys.path.insert(0, '.')
import numpy as np
import paper_2106_15214_b200 as bn
from paper_2106_15214_b200 import synthetic, solver

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 18
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
beta = float(sys.argv[3]) if len(sys.argv) > 3 else 1.5
v = synthetic.config4(N=N, dtype=np.float32)
w0, h0 = synthetic.uniform_init(256, N, 12, seed=112)
ctx = solver.get_context(0, "fp32")
ctx.set_dense(v, 0.0)
ctx.set_factors(w0, h0)
cfg = bn.SolverConfig(beta=beta, rank=12, algorithm="jmm", tol=1e-300, kappa=0.0, max_outer_iters=iters)
ctx.begin(solver.make_params(cfg, 0.0, kkt=False), iters)
ctx.set_profiling(True)
ms = ctx.step_timed(iters)
pm, ns = ctx.pass_time()
done, _ = ctx.sync()
obj, _, _ = ctx.trace(done)
print(f"N={N} iters={iters} ms/iter={ms/iters:.3f} pass_ms={pm:.3f} ({ns} samples) GB/s={256*N*4/(pm*1e-3)/1e9:.1f} obj={obj[-1]:.6e} sched={ctx.schedule()}")
