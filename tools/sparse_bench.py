"""Config-5 sparse KL timing (CSR, K=64): iterations/s of the device loop."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_2106_15214_b200 as bn
from paper_2106_15214_b200 import synthetic

F = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
N = int(sys.argv[2]) if len(sys.argv) > 2 else 200000
its = int(sys.argv[3]) if len(sys.argv) > 3 else 5
t0 = time.time()
indptr, idx, vals, shape = synthetic.config5(F=F, N=N)
print(f"gen {time.time()-t0:.1f}s nnz={len(vals)}", flush=True)
import scipy.sparse as sp
csr = sp.csr_matrix((vals, idx, indptr), shape=shape)
w0, h0 = synthetic.uniform_init(F, N, 64, seed=164)
cfg = bn.SolverConfig(beta=1.0, rank=64, algorithm="jmm", kappa=0.0, tol=1e-300, max_outer_iters=its)
t0 = time.time()
r = bn.fit(csr, cfg, init=(w0, h0), dtype="fp32")
el = time.time() - t0
sec = [t.seconds for t in r.trace]
print(f"fit wall {el:.1f}s; loop seconds {sec[-1]:.4f} for {its} its -> {its/sec[-1]:.1f} it/s; obj {r.trace[-1].objective:.6e}")
