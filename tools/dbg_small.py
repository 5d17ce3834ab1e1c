"""First objectives of the fp32 fused pass vs the oracle on a small config-4-like case."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2106_15214_b200 as bn
from oracle import betanmf_oracle as O

F = int(sys.argv[1]) if len(sys.argv) > 1 else 256
N = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
beta = float(sys.argv[3]) if len(sys.argv) > 3 else 1.5
K, its = 12, 5
v = bn.synthetic_low_rank(F, N, K, noise=0.05, seed=3).astype(np.float32)
init = bn.init_factors(F, N, K, seed=1)
for algo in ("jmm", "bmm"):
    cfg = bn.SolverConfig(beta=beta, rank=K, algorithm=algo, max_outer_iters=its, tol=1e-300)
    r = bn.fit(v, cfg, init=init, dtype='fp32', kkt=False)
    w, h, obj, _, _ = O.run(v.astype(np.float64), beta, K, algo, tol=1e-300, max_outer_iters=its,
                            init=(init.w, init.h), kkt=False)
    got = np.array([x.objective for x in r.trace])
    print(algo, "got", got)
    print(algo, "ref", obj)
    print(algo, "W rel", np.max(np.abs(r.factors.w - w)) / np.max(np.abs(w)),
          "H rel", np.max(np.abs(r.factors.h - h)) / np.max(np.abs(h)))
