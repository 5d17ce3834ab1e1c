"""Event timeline of CTA 0 of the tcgen05 pass (libbnmf built with BNMF_TC_PROF=1)."""
import ctypes, os, sys
os.environ["BNMF_TC_PROF"] = "1"
sys.path.insert(0, '.')
import numpy as np
import paper_2106_15214_b200 as bn
from paper_2106_15214_b200 import synthetic, solver, _native

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
p0 = int(sys.argv[2]) if len(sys.argv) > 2 else 200
p1 = int(sys.argv[3]) if len(sys.argv) > 3 else 230
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
G = 148
buf = (ctypes.c_longlong * (G * 48 + 3 * 4096))()
n = lib.bnmf_tc_prof_read(buf, len(buf))
a = np.array(buf[:n], dtype=np.int64)
names = {1: "D issue", 2: "D issued", 3: "zfull wait", 4: "zfull ok", 5: "side issued", 6: "hn wait",
         7: "hn ok", 20: "H item", 21: "H dfull ok", 22: "Z written", 30: "W item", 31: "W dfull ok",
         50: "U2 remote arr", 40: "U1", 41: "U1 end", 42: "U2", 43: "U2 xfull ok", 44: "U2 end", 45: "U2 math done",
         46: "U2 wdone ok", 47: "U2 hn arrived", 48: "U1 acch ok", 49: "U2 lds done", 51: "fold end"}
ev = []
for w, role in ((1, "MMA"), (2, "EPI")):
    base = G * 48 + w * 4096
    cnt = int(a[base + 4095])
    for x in a[base:base + cnt]:
        t, e, pos = int(x) >> 16, (int(x) >> 10) & 63, int(x) & 1023
        ev.append((t, role, names.get(e, str(e)), pos))
ev.sort()
# time window: from the first event of item p0 to the last event of item p1
win = [t for t, role, nm, pos in ev if nm in ("H item", "W item", "Z written") and p0 <= pos <= p1]
ta, tb = min(win), max(win)
for t, role, nm, pos in ev:
    if ta <= t <= tb:
        print(f"{t - ta:8d}  {role:3s}  {nm:12s} {'item' if nm not in ('U2 xfull ok',) else 'blk '} {pos}")
