"""Wait-cycle breakdown of the second-generation tcgen05 pass (lib built with BNMF_TC_PROF):
    BNMF_LIB=variants/libprof.so python tools/tc2_prof.py [N]"""
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
KKT = os.environ.get('KKT', '0') == '1'   # KKT=1: the counters of the H-side KKT pass (the last launch)
ctx.begin(solver.make_params(cfg, 0.0, kkt=KKT), 2)
ctx.step_timed(2)
ctx.sync()
kind, grid, cl, f0 = ctx.pass_info()
lib = _native.load()
buf = (ctypes.c_longlong * (grid * 288))()
n = lib.bnmf_tc_prof_read(buf, grid * 288)
NT = int(os.environ.get('BNMF_TC2_NT', '4'))
NW = 4 * NT + 7
a = np.array(buf[:grid * 12 * NW], dtype=np.int64).reshape(grid, NW, 12)
roles = {
    0: ("TMA", {0: "empty"}),
    1: ("Vt issuer", {0: "hp", 1: "hn", 2: "dfree"}),
    2: ("side issuer", {0: "zfull", 1: "accfree", 2: "accwfree"}),
    3: ("team0 q3", {0: "dfull(H)", 1: "dfull(W)", 2: "full(H)", 3: "full(W)", 4: "zfree", 5: "H items", 6: "W items", 7: "  H: stage wait + x loads", 8: "  H: tile wait + tcgen05.ld", 9: "  H: Z arithmetic + stores (incl. zfree)", 10: "  H: wait::st + fence + arrive"}),
    7: ("team1 q3", {0: "dfull(H)", 1: "dfull(W)", 2: "full(H)", 3: "full(W)", 4: "zfree", 5: "H items", 6: "W items"}),
    4 * NT - 1: ("last team q3", {0: "dfull(H)", 1: "dfull(W)", 2: "full(H)", 3: "full(W)", 4: "zfree", 5: "H items", 6: "W items"}),
    NW - 4: ("U team q3", {0: "hpfree", 1: "acch", 2: "xempty", 3: "xfull", 4: "wdone", 5: "accw", 6: "  acch->sends issued", 7: "acch->hn chain (incl. xempty/xfull/wdone waits)", 8: "  acch->AccH read", 9: "  acch->ratio done", 10: "  acch->peer partial added"}),
}
print(f"grid {grid}, N {N}")
for w, (name, cats) in roles.items():
    tot = a[:, w, 11].mean()
    print(f"{name}: total {tot/1e3:.1f} kcyc")
    for c, nm in cats.items():
        print(f"    {nm:10s} {a[:, w, c].mean()/1e3:9.1f} kcyc ({100*a[:, w, c].mean()/tot:5.1f}%)")
