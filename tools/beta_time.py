"""Pass time of the single-read tcgen05 kernel per beta class on a config-4 prefix."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2106_15214_b200 as bn
from paper_2106_15214_b200 import synthetic, solver
N = 1 << 20
v = synthetic.config4(N=N, dtype=np.float32)
w0, h0 = synthetic.uniform_init(256, N, 12, seed=112)
ctx = solver.get_context(0, "fp32")
ctx.set_dense(v, 0.0)
for beta in (0.0, 0.5, 1.0, 1.5, 2.0):
    ctx.set_factors(w0, h0)
    cfg = bn.SolverConfig(beta=beta, rank=12, algorithm="jmm", tol=1e-300, kappa=0.0, max_outer_iters=20)
    ctx.begin(solver.make_params(cfg, 0.0, kkt=False), 20)
    ctx.step(4)
    ms = ctx.step_timed(16)
    ctx.sync()
    print(f"beta={beta}: {ms / 16:.3f} ms per iteration at N = 2^20 ({256 * N * 4 / (ms / 16 * 1e-3) / 1e9:.0f} GB/s)")
