import sys; sys.path.insert(0, ".")
import numpy as np, paper_2106_15214_b200 as bn
from paper_2106_15214_b200 import synthetic as syn
for name, gen, K, beta in (("cfg3", syn.config3, 20, 0.0), ("cfg2", syn.config2, 32, 2.0)):
    v = gen().astype(np.float32); F, N = v.shape
    w0, h0 = syn.uniform_init(F, N, K, seed=100 + K)
    c = bn.SolverConfig(beta=beta, rank=K, algorithm="jmm", tol=1e-300, max_outer_iters=12)
    runs = [bn.fit(v, c, init=(w0, h0), dtype="fp32", kkt=True) for _ in range(3)]
    o = [np.array([r.objective for r in x.trace]) for x in runs]
    k = [np.array([[r.kkt_w, r.kkt_h] for r in x.trace]) for x in runs]
    print(name, "obj equal", np.array_equal(o[0], o[1]), np.array_equal(o[0], o[2]),
          "W equal", np.array_equal(runs[0].factors.w, runs[1].factors.w),
          "kkt equal", np.array_equal(k[0], k[1]), np.array_equal(k[0], k[2]))
    print(o[0][:4] - o[1][:4], o[0][:4] - o[2][:4])
