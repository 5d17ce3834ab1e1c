import os, sys
sys.path.insert(0, '.')
import numpy as np
import paper_2106_15214_b200 as bn
rng = np.random.default_rng(3)
for (f, n, k, beta) in [(300, 400, 100, 1.0), (700, 90, 128, 0.0), (129, 3000, 64, 1.5), (1000, 33, 5, 1.0)]:
    v = rng.gamma(1.0, 1.0, (f, 8)) @ rng.gamma(1.0, 1.0, (8, n)) + 1e-2
    w0 = rng.uniform(0.1, 1, (f, k)); h0 = rng.uniform(0.1, 1, (k, n))
    cfg = bn.SolverConfig(beta=beta, rank=k, algorithm="jmm", tol=1e-300, max_outer_iters=8)
    outs = []
    for cs in ("1", None):
        if cs: os.environ["BNMF_HSIDE_CLUSTER"] = cs
        else: os.environ.pop("BNMF_HSIDE_CLUSTER", None)
        r = bn.fit(v, cfg, init=(w0, h0))
        outs.append((np.array([t.objective for t in r.trace]), r.factors.w, r.factors.h, np.array([[t.kkt_w, t.kkt_h] for t in r.trace])))
    rel = lambda a, b: float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))
    print(f, n, k, beta, "obj", rel(outs[1][0], outs[0][0]), "w", rel(outs[1][1], outs[0][1]), "h", rel(outs[1][2], outs[0][2]), "kkt", rel(outs[1][3], outs[0][3]))
