"""200-iteration fp32 objective error of the fused tcgen05 pass vs the fp64
oracle (north_star: <= 1e-4 relative over 200 iterations, monotone)."""
import os, sys, numpy as np
sys.path.insert(0, '.')
import paper_2106_15214_b200 as bn
from oracle import betanmf_oracle as O

its = int(os.environ.get("ITS", "200"))
shapes = [(20, 130, 3), (64, 96, 4), (200, 2000, 8), (256, 4096, 12)]
betas = [float(b) for b in sys.argv[1].split(',')] if len(sys.argv) > 1 else [1.5, 1.0, 0.0, 2.0, 0.5]
worst = 0.0
for (F, N, K) in shapes:
    v = bn.synthetic_low_rank(F, N, K, noise=0.05, seed=3).astype(np.float32)
    init = bn.init_factors(F, N, K, seed=1)
    for beta in betas:
        for algo in ('jmm', 'bmm'):
            cfg = bn.SolverConfig(beta=beta, rank=K, algorithm=algo, max_outer_iters=its, tol=1e-300)
            r = bn.fit(v, cfg, init=init, dtype='fp32', kkt=False)
            _, _, obj, _, _ = O.run(v.astype(np.float64), beta, K, algo, tol=1e-300,
                                   max_outer_iters=its, init=(init.w, init.h), kkt=False)
            got = np.array([x.objective for x in r.trace])
            rel = np.abs(got - obj) / np.abs(obj)
            mono = bool(np.all(got[1:] <= got[:-1] * (1 + 1e-6)))
            worst = max(worst, rel.max())
            print(f"F{F} N{N} K{K} beta {beta} {algo}: max rel {rel.max():.2e} (it {rel.argmax()}) "
                  f"final {rel[-1]:.2e} monotone {mono}", flush=True)
print("worst", worst)
