"""Bring-up check of the tcgen05 fused pass against the oracle on small shapes
(cluster split F > 128, ragged F and N, every beta class, JMM and BMM)."""
import sys, time, numpy as np
sys.path.insert(0, '.')
import paper_2106_15214_b200 as bn
from oracle import betanmf_oracle as O

shapes = [(64, 96, 4), (200, 300, 12), (256, 1000, 12), (140, 257, 5), (20, 130, 3)]
betas = [float(b) for b in sys.argv[1].split(',')] if len(sys.argv) > 1 else [1.5, 1.0, 2.0, 0.0, 0.5]
its = 6
worst = 0.0
for (F, N, K) in shapes:
    v = bn.synthetic_low_rank(F, N, K, noise=0.05, seed=3).astype(np.float32)
    init = bn.init_factors(F, N, K, seed=1)
    for beta in betas:
        for algo in ('jmm', 'bmm'):
            t = time.time()
            cfg = bn.SolverConfig(beta=beta, rank=K, algorithm=algo, max_outer_iters=its, tol=1e-300)
            r = bn.fit(v, cfg, init=init, dtype='fp32', kkt=False)
            w, h, obj, _, _ = O.run(v.astype(np.float64), beta, K, algo, tol=1e-300,
                                   max_outer_iters=its, init=(init.w, init.h), kkt=False)
            got = np.array([x.objective for x in r.trace])
            oe = np.max(np.abs(got - obj) / np.abs(obj))
            we = np.max(np.abs(r.factors.w - w) / (np.abs(w) + 1e-6))
            he = np.max(np.abs(r.factors.h - h) / (np.abs(h) + 1e-6))
            worst = max(worst, oe)
            print(f"F{F} N{N} K{K} beta {beta} {algo}: obj {oe:.2e} W {we:.2e} H {he:.2e}"
                  f"  ({time.time() - t:.1f}s) sched={r.schedule if hasattr(r, 'schedule') else ''}",
                  flush=True)
print("worst objective rel error", worst)
