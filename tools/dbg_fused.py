import sys, numpy as np
sys.path.insert(0, '.')
import paper_2106_15214_b200 as bn
from oracle import betanmf_oracle as O
np.set_printoptions(precision=6, linewidth=150)
v = bn.synthetic_low_rank(64, 96, 4, noise=0.05, seed=3)
init = bn.init_factors(64, 96, 4, seed=1)
for beta in (2.0, 1.5):
  for algo in ('jmm', 'bmm'):
    for its in (1, 2, 3):
        cfg = bn.SolverConfig(beta=beta, rank=4, algorithm=algo, max_outer_iters=its, tol=1e-300)
        r = bn.fit(v.astype(np.float32), cfg, init=init, dtype='fp32', kkt=False)
        w, h, obj, _, _ = O.run(v.astype(np.float32).astype(np.float64), beta, 4, algo, tol=1e-300, max_outer_iters=its, init=(init.w, init.h), kkt=False)
        got = np.array([t.objective for t in r.trace])
        print(beta, algo, its, 'obj', got, obj, 'Werr %.2e Herr %.2e' % (np.max(np.abs(r.factors.w-w)/w), np.max(np.abs(r.factors.h-h)/h)))
