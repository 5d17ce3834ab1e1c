"""North-star fp32 gate fixtures: 200-iteration objective traces of the
REFERENCE ``betanmf`` package on the benchmarked shapes.

Run in the build container only (imports /root/reference/pkg/src):

    python tests/golden/gen_golden_gate.py [case ...]

Writes tests/golden/gate.npz: for every case and algorithm the reference's 200
objectives, its KKT residuals and the final W (small: F x K), computed in fp64
on the fp32-rounded V with the injected Uniform(0,1) init (SURVEY.md §8d
"correctness gates": objective within 1e-4 relative over 200 iterations).

Cases
  cfg2     config 2 at full size (1024 x 8192, K = 32, beta = 2)
  cfg3     config 3 at full size (1025 x 16384, K = 20, beta = 0, kappa auto)
  cfg4s    config 4, the first 16484 columns (129 column blocks, the last one
           ragged): with BNMF_TC_MAX_CLUSTERS=2 each CTA cluster of the tcgen05
           pass walks 64-65 blocks (TMEM folds, ring wraps, block interleave)
  cfg4b    a config-4-like shape with an uneven row split (200 x 8292, K = 16,
           beta = 0.5: the general-beta epilogue)
  cfg4k    256 x 8292, K = 12, beta = 1 (all-ones denominator path), kappa = 0
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

from gen_golden import run_ref  # noqa: E402
from paper_2106_15214_b200 import synthetic  # noqa: E402

ITERS = 200

CASES = {
    # name: (V generator, K, beta, kappa)
    "cfg2": (lambda: synthetic.config2(), 32, 2.0, None),
    "cfg3": (lambda: synthetic.config3(), 20, 0.0, None),
    "cfg4s": (lambda: synthetic.config4(N=16484), 12, 1.5, 0.0),
    "cfg4b": (lambda: synthetic.config4(F=200, N=8292, K=16, seed=41), 16, 0.5, None),
    "cfg4k": (lambda: synthetic.config4(N=8292, seed=42), 12, 1.0, 0.0),
}


def main(argv):
    path = os.path.join(HERE, "gate.npz")
    out = dict(np.load(path)) if os.path.exists(path) else {}
    for name in (argv or list(CASES)):
        gen, K, beta, kappa = CASES[name]
        v = gen().astype(np.float32).astype(np.float64)
        F, N = v.shape
        w0, h0 = synthetic.uniform_init(F, N, K, seed=100 + K)
        for algo in ("jmm", "bmm"):
            t0 = time.time()
            w, h, obj, kkt, term = run_ref(
                v, init=(w0, h0), beta=beta, rank=K, algorithm=algo, kappa=kappa,
                max_outer_iters=ITERS, tol=1e-300)
            out[f"{name}_{algo}/obj"] = obj
            out[f"{name}_{algo}/kkt"] = kkt
            out[f"{name}_{algo}/w"] = w
            print(name, algo, f"{time.time() - t0:.1f}s", obj[0], obj[-1], flush=True)
        out[f"{name}/vsum"] = np.array(float(v.sum()))
        out[f"{name}/shape"] = np.array(v.shape)
        np.savez_compressed(path, **out)


if __name__ == "__main__":
    main(sys.argv[1:])
