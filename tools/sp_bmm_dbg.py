"""Per-iteration relative objective error of the sparse path vs the oracle restatement."""
import os, sys
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import numpy as np, scipy.sparse as sp
import paper_2106_15214_b200 as bn
from paper_2106_15214_b200 import synthetic
from oracle import betanmf_oracle as O
algo = sys.argv[1] if len(sys.argv) > 1 else "bmm"
indptr, idx, vals, shape = synthetic.config5(F=2000, N=400, density=0.1, seed=55)
csr = sp.csr_matrix((vals, idx, indptr), shape=shape)
w0, h0 = synthetic.uniform_init(shape[0], shape[1], 16, seed=116)
cfg = bn.SolverConfig(beta=1.0, rank=16, algorithm=algo, kappa=0.0, tol=1e-300, max_outer_iters=30)
r = bn.fit(csr, cfg, init=(w0, h0), dtype="fp32")
_, _, obj, _ = O.run_sparse_kl(csr.astype(np.float64), 16, algo, max_outer_iters=30, init=(w0, h0))
got = np.array([t.objective for t in r.trace])
np.set_printoptions(precision=2, linewidth=200)
print(algo, np.abs(got / obj - 1))
