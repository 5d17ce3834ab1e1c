"""Generate the golden fixtures by running the REFERENCE ``betanmf`` package.

Run in the build container only (it imports /root/reference/pkg/src, which
does not exist on the GPU box):

    python tests/golden/gen_golden.py

Outputs (committed, small):
  tests/golden/fits.npz     whole fits: W, H, objective and KKT traces, for
                            every beta of the reference grid x {jmm, bmm} and
                            the kappa / sub-iteration / gamma variants
  tests/golden/kernels.npz  single update-kernel outputs on random instances
  tests/golden/configs.npz  the BASELINE configs (1 at full size, 2-4 as column
                            prefixes, 5 as a densified small sparse matrix) with
                            the injected Uniform(0,1) init

The init is injected exactly as SURVEY.md §8c describes: the reference resolves
``init_factors`` as a module global at solver.py:293, so it is monkeypatched.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import betanmf  # noqa: E402  (the reference)
import betanmf.solver as ref_solver  # noqa: E402
from betanmf import updates as ref_updates  # noqa: E402
from betanmf.majorizer import MajorizerAnchor  # noqa: E402

from paper_2106_15214_b200 import synthetic  # noqa: E402

BETA_GRID = (-0.5, 0.0, 0.5, 1.0, 1.5, 2.0, 3.0)


def run_ref(v, init=None, **cfg):
    """Run the reference fit, optionally with an injected init."""
    config = betanmf.SolverConfig(**cfg)
    saved = ref_solver.init_factors
    if init is not None:
        w0, h0 = init
        ref_solver.init_factors = lambda F, N, K, seed: betanmf.FactorPair(
            w0.copy(), h0.copy())
    try:
        res = betanmf.fit(v, config)
    finally:
        ref_solver.init_factors = saved
    obj = np.array([r.objective for r in res.trace])
    kkt = np.array([[r.kkt_w, r.kkt_h] for r in res.trace])
    return res.factors.w, res.factors.h, obj, kkt, res.termination.value


def fits():
    out = {}
    cases = []
    v_small = betanmf.synthetic_low_rank(12, 10, 3, noise=0.1, seed=2)
    for beta in BETA_GRID:
        for algo in ("jmm", "bmm"):
            cases.append((f"grid_b{beta}_{algo}", v_small,
                          dict(beta=beta, rank=3, algorithm=algo, seed=1,
                               kappa=0.0, max_outer_iters=40, tol=1e-300)))
    v_mid = betanmf.synthetic_low_rank(37, 29, 5, noise=0.05, seed=11)
    for beta in (0.0, 1.0, 1.5, 2.0):
        for algo in ("jmm", "bmm"):
            cases.append((f"mid_b{beta}_{algo}", v_mid,
                          dict(beta=beta, rank=5, algorithm=algo, seed=7,
                               max_outer_iters=25, tol=1e-300)))
    # variants: kappa auto with zeros, explicit kappa, sub-iterations, gamma=1,
    # convergence stop, exact fit, rank 1 / ragged shapes
    vz = v_mid.copy()
    vz[::3, ::4] = 0.0
    cases += [
        ("kappa_auto_b0_jmm", vz, dict(beta=0.0, rank=4, algorithm="jmm", seed=3,
                                        max_outer_iters=20, tol=1e-300)),
        ("kappa_auto_b05_bmm", vz, dict(beta=0.5, rank=4, algorithm="bmm", seed=3,
                                         max_outer_iters=20, tol=1e-300)),
        ("kappa_0.3_b1.5_jmm", v_mid, dict(beta=1.5, rank=4, algorithm="jmm", seed=4,
                                           kappa=0.3, max_outer_iters=20, tol=1e-300)),
        ("kappa_0.3_b2_bmm", v_mid, dict(beta=2.0, rank=4, algorithm="bmm", seed=4,
                                         kappa=0.3, max_outer_iters=20, tol=1e-300)),
        ("sub3_b1.5_jmm", v_mid, dict(beta=1.5, rank=4, algorithm="jmm", seed=5,
                                      sub_iters=3, max_outer_iters=15, tol=1e-300)),
        ("sub3_b0_jmm", v_mid, dict(beta=0.0, rank=4, algorithm="jmm", seed=5,
                                    sub_iters=3, max_outer_iters=15, tol=1e-300)),
        ("sub2x3_b1_bmm", v_mid, dict(beta=1.0, rank=4, algorithm="bmm", seed=5,
                                      sub_iters_w=2, sub_iters_h=3,
                                      max_outer_iters=15, tol=1e-300)),
        ("gamma1_b0_jmm", v_mid, dict(beta=0.0, rank=4, algorithm="jmm", seed=6,
                                      heuristic_gamma_one=True,
                                      max_outer_iters=20, tol=1e-300)),
        ("gamma1_b3_bmm", v_mid, dict(beta=3.0, rank=4, algorithm="bmm", seed=6,
                                      heuristic_gamma_one=True,
                                      max_outer_iters=20, tol=1e-300)),
        ("converge_b1_jmm", v_mid, dict(beta=1.0, rank=5, algorithm="jmm", seed=2,
                                        tol=1e-4, max_outer_iters=5000)),
        ("converge_b2_bmm", v_mid, dict(beta=2.0, rank=5, algorithm="bmm", seed=2,
                                        tol=1e-4, max_outer_iters=5000)),
        ("rank1_b1_jmm", v_mid[:7, :3], dict(beta=1.0, rank=1, algorithm="jmm",
                                            seed=9, max_outer_iters=10, tol=1e-300)),
        ("ragged_b1.5_bmm", betanmf.synthetic_low_rank(133, 67, 7, noise=0.1, seed=3),
         dict(beta=1.5, rank=7, algorithm="bmm", seed=2, max_outer_iters=12,
              tol=1e-300)),
        ("ragged_b0.5_jmm", betanmf.synthetic_low_rank(133, 67, 7, noise=0.1, seed=3),
         dict(beta=0.5, rank=7, algorithm="jmm", seed=2, max_outer_iters=12,
              tol=1e-300)),
    ]
    init = betanmf.init_factors(5, 4, 2, seed=3)
    cases.append(("exact_fit_b2_jmm", init.w @ init.h,
                  dict(beta=2.0, rank=2, algorithm="jmm", seed=3)))
    names = []
    for name, v, cfg in cases:
        w, h, obj, kkt, term = run_ref(v, **cfg)
        names.append(name)
        out[f"{name}/v"] = v
        out[f"{name}/w"] = w
        out[f"{name}/h"] = h
        out[f"{name}/obj"] = obj
        out[f"{name}/kkt"] = kkt
        out[f"{name}/term"] = np.array(term)
        cfg_s = repr(sorted(cfg.items()))
        out[f"{name}/cfg"] = np.array(cfg_s)
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "fits.npz"), **out)
    print("fits:", len(names))


def kernels():
    rng = np.random.default_rng(20240901)
    out = {}
    n = 0
    for beta in BETA_GRID:
        for t in range(3):
            v = rng.uniform(0.1, 3.0, size=(6, 5))
            wt = rng.uniform(0.1, 2.0, size=(6, 3))
            ht = rng.uniform(0.1, 2.0, size=(3, 5))
            hc = rng.uniform(0.1, 2.0, size=(3, 5))
            wc = rng.uniform(0.1, 2.0, size=(6, 3))
            kappa = 0.0 if t < 2 else 0.25
            anchor = MajorizerAnchor.from_factors(wt, ht, kappa=kappa)
            vs = v + kappa
            key = f"k{n}"
            out[f"{key}/beta"] = np.array(beta)
            out[f"{key}/kappa"] = np.array(kappa)
            for nm, arr in (("v", v), ("wt", wt), ("ht", ht), ("hc", hc), ("wc", wc)):
                out[f"{key}/{nm}"] = arr
            out[f"{key}/jmm_w"] = ref_updates.jmm_update_w(vs, anchor, hc, beta)
            out[f"{key}/jmm_h"] = ref_updates.jmm_update_h(vs, anchor, wc, beta)
            out[f"{key}/bmm_w"] = ref_updates.bmm_update_w(vs, wc, hc, beta, kappa=kappa)
            out[f"{key}/bmm_h"] = ref_updates.bmm_update_h(vs, wc, hc, beta, kappa=kappa)
            out[f"{key}/obj"] = np.array(betanmf.objective(
                betanmf.DataMatrix(v, kappa), betanmf.FactorPair(wc, hc), beta))
            kr = betanmf.kkt_residuals(betanmf.DataMatrix(v, kappa),
                                       betanmf.FactorPair(wc, hc), beta)
            out[f"{key}/kkt"] = np.array([kr.res_w, kr.res_h])
            n += 1
    out["count"] = np.array(n)
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **out)
    print("kernels:", n)


def configs(only_sparse=False):
    """BASELINE configs through the reference, fp64, injected U(0,1) init.

    fp32 configs are run on the fp32-rounded V (SURVEY.md §8d correctness gates).
    ``only_sparse`` regenerates just the cfg5p entries (after a change of the
    config-5 generator) and keeps the rest of configs.npz.
    """
    path = os.path.join(HERE, "configs.npz")
    out = dict(np.load(path)) if only_sparse else {}
    specs = [
        # name, V generator, K, beta, iters, kappa(None=auto), fp32?
        ("cfg1", lambda: synthetic.config1(), 49, 1.0, 200, None, False),
        ("cfg2p", lambda: synthetic.config2(F=1024, N=1024, K=32), 32, 2.0, 60, None, True),
        ("cfg3p", lambda: synthetic.config3(F=1025, N=1024, K=20), 20, 0.0, 60, None, True),
        ("cfg4p", lambda: synthetic.config4(N=4096), 12, 1.5, 60, 0.0, True),
    ]
    for name, gen, K, beta, iters, kappa, fp32 in ([] if only_sparse else specs):
        v = gen()
        if fp32:
            v = v.astype(np.float32).astype(np.float64)
        F, N = v.shape
        w0, h0 = synthetic.uniform_init(F, N, K, seed=100 + K)
        for algo in ("jmm", "bmm"):
            if name == "cfg1" and algo == "bmm":
                its = 50
            else:
                its = iters
            w, h, obj, kkt, term = run_ref(
                v, init=(w0, h0), beta=beta, rank=K, algorithm=algo, kappa=kappa,
                max_outer_iters=its, tol=1e-300)
            out[f"{name}_{algo}/w"] = w
            out[f"{name}_{algo}/h"] = h
            out[f"{name}_{algo}/obj"] = obj
            out[f"{name}_{algo}/kkt"] = kkt
        out[f"{name}/vsum"] = np.array(float(v.sum()))
        out[f"{name}/shape"] = np.array(v.shape)
    # sparse KL stand-in: small config-5-like count matrix, densified for the
    # reference (kappa must be 0 explicitly)
    indptr, idx, vals, shape = synthetic.config5(F=2000, N=400, density=0.1, seed=55)
    import scipy.sparse as sp
    dense = sp.csr_matrix((vals.astype(np.float64), idx, indptr), shape=shape).toarray()
    w0, h0 = synthetic.uniform_init(shape[0], shape[1], 16, seed=116)
    for algo in ("jmm", "bmm"):
        w, h, obj, kkt, term = run_ref(dense, init=(w0, h0), beta=1.0, rank=16,
                                       algorithm=algo, kappa=0.0,
                                       max_outer_iters=30, tol=1e-300)
        out[f"cfg5p_{algo}/w"] = w
        out[f"cfg5p_{algo}/h"] = h
        out[f"cfg5p_{algo}/obj"] = obj
        out[f"cfg5p_{algo}/kkt"] = kkt
    out["cfg5p/nnz"] = np.array(idx.size)
    out["cfg5p/vsum"] = np.array(float(vals.astype(np.float64).sum()))
    np.savez_compressed(path, **out)
    print("configs written")


if __name__ == "__main__":
    if sys.argv[1:] == ["cfg5p"]:
        configs(only_sparse=True)
    else:
        fits()
        kernels()
        configs()
