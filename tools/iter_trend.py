"""Per-iteration time of the fused pass over a long run (trace seconds), to separate data-dependent
slow-downs from clock effects:  python tools/iter_trend.py [N] [iters]"""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2106_15214_b200 as bn
from paper_2106_15214_b200 import synthetic, solver

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 120
v = synthetic.config4(N=N, dtype=np.float32)
w0, h0 = synthetic.uniform_init(256, N, 12, seed=112)
ctx = solver.get_context(0, "fp32")
ctx.set_dense(v, 0.0)
cfg = bn.SolverConfig(beta=1.5, rank=12, algorithm="jmm", tol=1e-300, kappa=0.0, max_outer_iters=iters)
for rep in range(2):   # the second run restarts from the same factors right after the first
    ctx.set_factors(w0, h0)
    ctx.begin(solver.make_params(cfg, 0.0, kkt=False), iters)
    ms = ctx.step_timed(iters)
    done, _ = ctx.sync()
    obj, sec, _ = ctx.trace(done)
    d = np.diff(np.asarray(sec)) * 1e3
    print("ms/iter by decade:", " ".join(f"{d[i:i+10].mean():.3f}" for i in range(0, len(d), 10)))
    print(f"  first 20: {d[:20].mean():.3f} ms, from iteration 100 on (power-capped clocks): {d[100:].mean():.3f} ms")
w, h = ctx.factors()
h = np.asarray(h)
print("H: zeros %.3f, subnormal(fp32) %.4f, <1e-30 %.4f" % ((h == 0).mean(), ((h != 0) & (np.abs(h) < 1.18e-38)).mean(), (np.abs(h) < 1e-30).mean()))
