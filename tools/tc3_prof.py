"""Wait-cycle breakdown of the tcgen05 pass pair on config 4 (lib built with -DBNMF_TC_PROF):
    BNMF_TC_PAIR=1 BNMF_LIB=variants/libprof.so python tools/tc3_prof.py [N]
The buffer holds the counters of the LAST pass_tc3 launch (the W pass)."""
import ctypes, os, sys
os.environ["BNMF_TC_PROF"] = "1"
sys.path.insert(0, '.')
import numpy as np
import paper_2106_15214_b200 as bn
from paper_2106_15214_b200 import synthetic, solver, _native

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
mode = sys.argv[2] if len(sys.argv) > 2 else "W"
v = synthetic.config4(N=N, dtype=np.float32)
w0, h0 = synthetic.uniform_init(256, N, 12, seed=112)
ctx = solver.get_context(0, "fp32")
ctx.set_dense(v, 0.0)
ctx.set_factors(w0, h0)
cfg = bn.SolverConfig(beta=1.5, rank=12, algorithm="jmm", tol=1e-300, kappa=0.0, max_outer_iters=2)
ctx.begin(solver.make_params(cfg, 0.0, kkt=False), 2)
ctx.step_timed(2)
ctx.sync()
kind, grid, cl, f0 = ctx.pass_info()
lib = _native.load()
NW = 23
buf = (ctypes.c_longlong * (grid * NW * 12))()
n = lib.bnmf_tc_prof_read(buf, grid * NW * 12)
a = np.array(buf[:grid * NW * 12], dtype=np.int64).reshape(grid, NW, 12)
names = {0: ("TMA", {0: "empty"}), 1: ("Vt issuer", {0: "op", 1: "dfree"}),
         2: ("side issuer", {0: "zfull", 1: "accfree", 2: "issue"}),
         3: ("team0 q3", {0: "dfull", 1: "zfree", 2: "full"}), 7: ("team1 q3", {0: "dfull", 1: "zfree", 2: "full"}),
         19: ("U team q3", {0: "opfree", 1: "acc"})}
print(f"grid {grid}, N {N}, last launch = {mode} pass")
for w, (name, cats) in names.items():
    tot = a[:, w, 11].mean()
    print(f"{name}: total {tot/1e3:.1f} kcyc")
    for c, nm in cats.items():
        print(f"    {nm:10s} {a[:, w, c].mean()/1e3:9.1f} kcyc ({100*a[:, w, c].mean()/max(tot,1):5.1f}%)")
