"""Wait-cycle breakdown of the tcgen05 fused pass (BNMF_TC_PROF=1 build-free knob)."""
import ctypes, os, sys
os.environ["BNMF_TC_PROF"] = "1"
sys.path.insert(0, '.')
import numpy as np
import paper_2106_15214_b200 as bn
from paper_2106_15214_b200 import synthetic, solver, _native

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
v = synthetic.config4(N=N, dtype=np.float32)
w0, h0 = synthetic.uniform_init(256, N, 12, seed=112)
ctx = solver.get_context(0, "fp32")
ctx.set_dense(v, 0.0)
ctx.set_factors(w0, h0)
cfg = bn.SolverConfig(beta=1.5, rank=12, algorithm="jmm", tol=1e-300, kappa=0.0, max_outer_iters=2)
ctx.begin(solver.make_params(cfg, 0.0, kkt=False), 2)
ctx.step_timed(2)
ctx.sync()
lib = _native.load()
buf = (ctypes.c_longlong * (148 * 48))()
n = lib.bnmf_tc_prof_read(buf, 148 * 48)
a = np.array(buf[:n], dtype=np.int64).reshape(-1, 48)
names = {0: "prod: empty", 11: "prod: total", 12: "mma: dempty",
         13: "mma: hn", 14: "mma: hp", 15: "mma: zfull", 16: "mma: accfree", 17: "mma: accwfree", 18: "mma: dempty(DL)", 19: "mma: side issue", 23: "mma: total",
         24: "epi: dfull(H)", 25: "epi: full(H)", 26: "epi: dfull(W)", 27: "epi: acch", 28: "epi: xempty",
         29: "epi: xfull", 30: "epi: zempty+wdone", 31: "epi: accw", 32: "epi: U1", 33: "epi: U2", 34: "epi: fold total",
         35: "epi: total"}
tot = a[:, 35].mean()
for k, nm in names.items():
    print(f"{nm:18s} mean {a[:, k].mean()/1e3:10.1f} kcyc  ({100*a[:, k].mean()/tot:5.1f}% of epilogue total)")
