#!/usr/bin/env python
"""Benchmark: beta-NMF joint-MM outer iterations/s on B200 (BASELINE.json metric).

Default workload (N=1): BASELINE config 4 -- beta = 1.5 joint-MM, fp32,
V 256 x 4,194,304 (4.29 GB, far larger than the 126 MB L2), K = 12 -- the
largest single-GPU configuration and the one the metric's 1-8 GPU scaling is
quoted on.  A "step" is one outer iteration (solver.py:301-319): update of W and
H, objective of the new iterate, normalisation.  Under torchrun the columns are
sharded across ranks (strong scaling of the fixed 4.2M-column problem).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1..4]
    python bench.py --impl reference ...   # CPU reference arm (oracle port)

Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "beta-NMF joint-MM outer iterations/s (V-pass HBM GB/s in roofline)"

CONFIGS = {
    # name: F, N, K, beta, dtype, kappa
    1: dict(F=361, N=2429, K=49, beta=1.0, dtype="fp64", kappa=0.0),
    2: dict(F=1024, N=8192, K=32, beta=2.0, dtype="fp32", kappa=0.0),
    3: dict(F=1025, N=16384, K=20, beta=0.0, dtype="fp32", kappa=None),
    4: dict(F=256, N=4194304, K=12, beta=1.5, dtype="fp32", kappa=0.0),
    # sparse KL (CSR, 0.05 % density -> 10^8 nonzeros, Zipf(1.1) columns), row-sharded
    5: dict(F=1000000, N=200000, K=64, beta=1.0, dtype="fp32", kappa=0.0, density=5e-4),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4, choices=sorted(CONFIGS))
    ap.add_argument("--algo", default="jmm", choices=["jmm", "bmm"])
    ap.add_argument("--schedule", default="auto", choices=["auto", "reference", "fused"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def make_data(cfg_id, n0, n1, dtype):
    from paper_2106_15214_b200 import synthetic as syn
    c = CONFIGS[cfg_id]
    npdt = np.float32 if dtype == "fp32" else np.float64
    if cfg_id == 4:
        return syn.config4(F=c["F"], N=c["N"], K=c["K"], dtype=npdt, col_range=(n0, n1))
    gen = {1: syn.config1, 2: syn.config2, 3: syn.config3}[cfg_id]
    v = gen(F=c["F"], N=c["N"], K=c["K"])
    return np.ascontiguousarray(v[:, n0:n1]).astype(npdt)


def make_init(cfg_id, n0, n1):
    from paper_2106_15214_b200 import synthetic as syn
    c = CONFIGS[cfg_id]
    w0, h0 = syn.uniform_init(c["F"], c["N"], c["K"], seed=100 + c["K"])
    return w0, np.ascontiguousarray(h0[:, n0:n1])


# measured tensor peaks (tools/tensor_peaks.cu, profiles/r02_tensor_peaks.txt): the fp32 passes
# run 3xTF32 products on tcgen05 (a third of the dense TF32 rate), the fp64 kernels run DMMA
TENSOR_PEAK_TFLOPS = {"fp32": 1114.4 / 3.0, "fp64": 37.11}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), float(d.get("bf16_tflops", 1590.0)), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """Samples SM clocks and throttle reasons through NVML during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            pass
        self._stop = threading.Event()

    def _loop(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons - {"gpu_idle"}), "samples": len(self.samples)}


def _import_reference():
    """The unmodified reference package installed under baseline/_ref (pip
    --target of /root/reference/pkg; git-ignored, travels to the GPU box), or
    None when it is absent."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "betanmf")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        import betanmf
        import betanmf.solver
        return betanmf
    except Exception:
        return None


def reference_sample_cols(cfg_id):
    """Columns of the bounded CPU sample: a 65536-column prefix of config 4
    (1/64 of the workload; columns are independent given W, so the time per
    iteration is linear in N), the whole matrix otherwise."""
    c = CONFIGS[cfg_id]
    return min(c["N"], 65536) if cfg_id == 4 else c["N"]


def time_reference(cfg_id, algo, warmup, steps):
    """Time the reference's own CPU loop on the bounded sample; returns
    (seconds per outer iteration on the sample, info dict)."""
    c = CONFIGS[cfg_id]
    from threadpoolctl import threadpool_limits, threadpool_info

    cores = os.cpu_count() or 1
    n_sample = reference_sample_cols(cfg_id)
    scale = c["N"] / n_sample
    v = make_data(cfg_id, 0, n_sample, c["dtype"]).astype(np.float64)
    w0, h0 = make_init(cfg_id, 0, n_sample)
    iters = warmup + steps
    ref = _import_reference()
    t_wall = time.perf_counter()
    with threadpool_limits(limits=cores):
        blas_threads = max([d.get("num_threads", 0) for d in threadpool_info()] or [0])
        if ref is not None:
            kind = "reference"
            saved = ref.solver.init_factors
            ref.solver.init_factors = lambda F, N, K, seed: ref.FactorPair(w0.copy(), h0.copy())
            try:
                cfg = ref.SolverConfig(beta=c["beta"], rank=c["K"], algorithm=algo,
                                       kappa=c["kappa"], tol=1e-300, max_outer_iters=iters)
                res = ref.fit(v, cfg)
            finally:
                ref.solver.init_factors = saved
            secs = np.array([r.seconds for r in res.trace])
            times = np.diff(np.concatenate([[0.0], secs]))[warmup:]
            what = "betanmf.fit (unmodified reference, baseline/_ref), TraceRow.seconds"
        else:
            kind = "port"
            from oracle import betanmf_oracle as O
            times = []
            w, h = w0, h0
            for i in range(iters):
                t0 = time.perf_counter()
                w, h, _, _, _ = O.run(v, c["beta"], c["K"], algo, kappa=c["kappa"],
                                      tol=1e-300, max_outer_iters=1, init=(w, h), kkt=False)
                if i >= warmup:
                    times.append(time.perf_counter() - t0)
            times = np.array(times)
            what = "numpy port of the reference loop (oracle/betanmf_oracle.py), perf_counter"
    wall = time.perf_counter() - t_wall
    dt = float(np.mean(times))
    sample = (f"{what}; fp64; {c['F']}x{n_sample} column prefix of {c['F']}x{c['N']} "
              f"(1/{scale:g} of the workload); each step = one outer iteration on the prefix, "
              f"measured {dt * 1e3:.1f} ms; value = 1 / (that x {scale:g})")
    return dt, dict(cores=cores, kind=kind, n_sample=n_sample, scale=scale, sample=sample,
                    wall_s=round(wall, 2), blas_threads=blas_threads)


def run_reference(args):
    """Reference arm: the reference's own CPU loop on the box's host cores.

    With baseline/_ref present this is the unmodified ``betanmf.fit``
    (run_jmm / run_bmm) with the bench's injected Uniform(0,1) init
    (monkeypatched ``init_factors``, as tests/golden/gen_golden.py does), timed
    by the reference's own loop timer (``TraceRow.seconds``: monotonic, KKT
    excluded, solver.py:302-312), BLAS on every host core; otherwise the
    numpy port in oracle/.  Each step is one outer iteration on the bounded
    sample (reference_sample_cols); ``ms_per_step`` is that measured time and
    ``value`` the iterations/s it implies for the full workload."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    dt, info = time_reference(args.config, args.algo, args.warmup, args.steps)
    val = 1.0 / (dt * info["scale"])
    out = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "iterations/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, world),
        "sample": {"n_cols": info["n_sample"], "scale_to_workload": info["scale"],
                   "ms_per_step_on_sample": dt * 1e3,
                   "ms_per_full_iteration": dt * info["scale"] * 1e3,
                   "wall_s": info["wall_s"], "blas_threads": info["blas_threads"]},
        "cpu_baseline": {"value": val, "unit": "iterations/s", "cores": info["cores"],
                         "kind": info["kind"], "sample": info["sample"]},
        "e2e": {"value": val, "unit": "iterations/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))


def workload_config(args, world):
    c = CONFIGS[args.config]
    return {"workload": f"config{args.config}: {args.algo} beta={c['beta']} {c['F']}x{c['N']} "
                        f"K={c['K']} {c['dtype']}",
            "F": c["F"], "N": c["N"], "K": c["K"], "beta": c["beta"], "algorithm": args.algo,
            "parallelism": f"N-columns x{world}", "l2": "inputs larger than L2"
            if c["F"] * c["N"] * (4 if c["dtype"] == "fp32" else 8) > 126e6
            else "input fits in L2 (no flush; iterations re-read V)"}


def run_sparse(args):
    """Config 5: the sparse KL path (CSR on the device, SDDMM at the nonzeros).

    value = device-timed iterations/s (kkt=False, like the dense configs); the roofline is the
    byte model of SURVEY.md §8(d): CSR index + value (8 B per nonzero), W~ read + W written,
    H~ read + H numerators written, over the measured HBM bandwidth, for the whole iteration
    (the path is several kernels; none dominates).  cpu_baseline = the scipy.sparse restatement
    of the reference loop (oracle.run_sparse_kl; the reference itself densifies and cannot
    ingest config 5) on a row prefix, scaled by rows."""
    rank, world, local = dist_env()
    if world > 1:
        raise SystemExit("bench.py --config 5 measures one GPU (row sharding is covered by "
                         "tests/test_parallel_gloo.py)")
    import scipy.sparse as sp
    import torch
    torch.cuda.set_device(local)
    import paper_2106_15214_b200 as bn
    from paper_2106_15214_b200 import solver, synthetic as syn
    c = CONFIGS[5]
    t0 = time.perf_counter()
    indptr, idx, vals, shape = syn.config5(F=c["F"], N=c["N"], density=c["density"])
    F, N = shape
    nnz = int(vals.size)
    gen_s = time.perf_counter() - t0
    w0, h0 = syn.uniform_init(F, N, c["K"], seed=100 + c["K"])
    csr = sp.csr_matrix((vals, idx, indptr), shape=shape)
    arrays, _ = solver.csr_with_csc_view(csr)
    config = bn.SolverConfig(beta=1.0, rank=c["K"], algorithm=args.algo, tol=1e-300, kappa=0.0,
                             max_outer_iters=args.warmup + args.steps + 1)
    ctx = solver.get_context(local, "fp32-sparse")
    ctx.set_csr(*arrays, (F, N))
    ctx.set_factors(w0, h0)
    ctx.begin(solver.make_params(config, 0.0, kkt=False, schedule="reference"),
              args.warmup + args.steps + 1)
    ctx.step(args.warmup)
    ctx.sync()
    clocks = ClockSampler(local)
    with clocks:
        ms = ctx.step_timed(args.steps)
    ctx.step(1)   # the trailing slot finishes the last iterate's trace row
    done, _ = ctx.sync()
    if done < args.warmup + args.steps:
        raise RuntimeError(f"only {done} iterations ran")
    obj, _, _ = ctx.trace(done)
    launches = ctx.launches_per_iter()
    value = args.steps / (ms / 1e3)
    hbm, _, peak_src = measured_peaks()
    bytes_iter = 8 * nnz + 8 * (F + 1) + 2 * F * c["K"] * 4 + 2 * N * c["K"] * 4
    achieved = bytes_iter / (ms / args.steps / 1e3) / 1e9
    out = {
        "metric": METRIC, "value": value, "unit": "iterations/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": f"config5: sparse KL {args.algo} {F}x{N} CSR nnz={nnz} K={c['K']} fp32",
                   "F": F, "N": N, "K": c["K"], "beta": 1.0, "algorithm": args.algo, "nnz": nnz,
                   "parallelism": "rows x1", "l2": "inputs larger than L2"},
        "schedule": "sparse", "gpu_launches": launches * args.steps,
        "roofline": {"bound": "hbm", "kernel": "sparse iteration (sp_pass_a + sp_pass_b* + sp_pass_c)",
                     "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": None, "peak_source": f"{peak_src} (MEASURED_PEAKS.json hbm_gbs)",
                     "algorithmic_bytes_per_launch": bytes_iter,
                     "bytes_model": "8 B per nonzero (CSR index + value) + indptr + W~ read + W "
                                    "written + H~ read + H numerators written (SURVEY.md 8d)"},
        "clocks": clocks.summary(), "final_objective": float(obj[done - 1]),
        "iterations_done": int(done), "generation_s": round(gen_s, 1),
    }
    if not args.no_cpu:
        from oracle import betanmf_oracle as O
        from threadpoolctl import threadpool_limits
        fs = 50000
        sub = csr[:fs].astype(np.float64)
        with threadpool_limits(limits=os.cpu_count() or 1):
            t0 = time.perf_counter()
            O.run_sparse_kl(sub, c["K"], args.algo, max_outer_iters=2, init=(w0[:fs], h0))
            dt = (time.perf_counter() - t0) / 2
        out["cpu_baseline"] = {
            "value": 1.0 / (dt * F / fs), "unit": "iterations/s", "cores": os.cpu_count() or 1,
            "kind": "port",
            "sample": f"scipy.sparse restatement of the reference loop (oracle.run_sparse_kl; the "
                      f"reference densifies and cannot ingest config 5); first {fs} of {F} rows "
                      f"({sub.nnz} nonzeros), 2 iterations, {dt * 1e3:.0f} ms each; value = 1 / "
                      f"(that x {F // fs})"}
    print(json.dumps(out))


def main():
    args = parse()
    if args.impl == "reference" and args.config != 5:
        run_reference(args)
        return
    if args.config == 5:
        if args.impl == "reference":
            raise SystemExit("the reference arm of config 5 is the cpu_baseline of the default arm")
        run_sparse(args)
        return
    rank, world, local = dist_env()
    import torch
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2106_15214_b200 as bn
    from paper_2106_15214_b200 import _native, parallel, solver

    c = CONFIGS[args.config]
    align = 65536 if args.config == 4 else 4
    n0, n1 = parallel.balanced_blocks(c["N"], world, align)[rank]
    v = make_data(args.config, n0, n1, c["dtype"])
    w0, h0 = make_init(args.config, n0, n1)
    config = bn.SolverConfig(beta=c["beta"], rank=c["K"], algorithm=args.algo, tol=1e-300,
                             kappa=c["kappa"], max_outer_iters=args.warmup + args.steps)
    kappa = parallel.resolve_kappa_global(v, c["beta"], c["kappa"]) if world > 1 else (
        c["kappa"] if c["kappa"] is not None else bn.default_kappa(v, c["beta"]))

    # ---- device-timed region: W warm-up + K timed iterations -------------
    ctx = solver.get_context(local, c["dtype"])
    if world > 1:
        solver._attach_comm(ctx, c["N"])
    ctx.set_dense(v, kappa)
    ctx.set_factors(w0, h0)
    ctx.begin(solver.make_params(config, kappa, kkt=False, schedule=args.schedule),
              args.warmup + args.steps)
    ctx.set_profiling(True)
    ctx.step(args.warmup)
    ctx.sync()
    if world > 1:
        torch.distributed.barrier()
    clocks = ClockSampler(local)
    with clocks:
        ms = ctx.step_timed(args.steps)
    pass_ms, pass_samples = ctx.pass_time()
    ctx.set_profiling(False)   # the e2e leg below runs without per-pass events
    done, _ = ctx.sync()
    if done != args.warmup + args.steps:
        raise RuntimeError(f"only {done} of {args.warmup + args.steps} iterations ran (the stop "
                           "rule fired); the timed region would include no-op slots")
    obj, _, _ = ctx.trace(done)
    launches = ctx.launches_per_iter()
    sched = ctx.schedule()
    ms_all = parallel.allreduce_scalars([ms, pass_ms], "max") if world > 1 else [ms, pass_ms]
    ms, pass_ms = float(ms_all[0]), float(ms_all[1])
    value = args.steps / (ms / 1e3)

    # ---- end to end: the public API on host buffers ----------------------
    e2e = None
    if not args.no_e2e:
        import torch
        vp = torch.from_numpy(v).pin_memory().numpy()
        cfg_e = bn.SolverConfig(beta=c["beta"], rank=c["K"], algorithm=args.algo, tol=1e-300,
                                kappa=kappa, max_outer_iters=args.steps)
        # one untimed warm-up call (first-call allocations, graph capture), like the W
        # warm-up steps of the device-timed region; the timed call then repeats every
        # host-side step: checks, H2D of V and the init, the iterations, D2H of W, H, trace
        cfg_w = bn.SolverConfig(beta=c["beta"], rank=c["K"], algorithm=args.algo, tol=1e-300,
                                kappa=kappa, max_outer_iters=max(1, args.warmup))
        bn.fit(vp, cfg_w, init=(w0, h0), dtype=c["dtype"], schedule=args.schedule,
               sharded=world > 1)
        # median of five timed calls: the host side (fresh fp64 result arrays, pageable
        # copies of the init and factors) varies by +-30 % from call to call, with outliers
        tes = []
        for _rep in range(5):
            if world > 1:
                torch.distributed.barrier()
            t0 = time.perf_counter()
            # the API default: kkt=True (trace rows carry the KKT residuals like the
            # reference's; they are computed by the fused KKT pass after each iteration)
            res = bn.fit(vp, cfg_e, init=(w0, h0), dtype=c["dtype"],
                         schedule=args.schedule, sharded=world > 1)
            _ = res.trace[-1].objective
            te = time.perf_counter() - t0
            tes.append(float(parallel.allreduce_scalars([te], "max")[0]) if world > 1 else te)
        te = statistics.median(tes)
        h2d = v.nbytes + w0.nbytes + h0.nbytes
        d2h = res.factors.w.nbytes + res.factors.h.nbytes + 24 * args.steps
        e2e = {"value": args.steps / te, "unit": "iterations/s",
               "h2d_bytes_per_step": int(h2d * world / args.steps),
               "d2h_bytes_per_step": int(d2h * world / args.steps),
               "note": "median of 5 default fit() calls (kkt=True) on pinned host V after one "
                       f"untimed warm-up call; each: upload, domain checks, {args.steps} "
                       "iterations with their KKT passes, download of W, H and trace",
               "calls_s": [round(t, 4) for t in tes]}

    if rank != 0:
        return
    hbm, _, peak_src = measured_peaks()
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tr = json.load(f).get(f"config{args.config}:{args.algo}:"
                                  f"{'fused_pass_tc' if sched == 'fused' else 'hside_pass'}")
        if tr and world == 1:
            traffic = tr["dram_bytes_per_launch"]
    except Exception:
        traffic = None
    esize = 4 if c["dtype"] == "fp32" else 8
    vbytes_local = c["F"] * (n1 - n0) * esize
    achieved = vbytes_local / (pass_ms / 1e3) / 1e9 if pass_ms > 0 else None
    roofline = {
        "bound": "hbm", "kernel": "fused_pass" if sched == "fused" else "hside_pass",
        "achieved": achieved, "peak": hbm, "unit": "GB/s",
        "frac": achieved / hbm if achieved else None, "traffic": traffic,
        "traffic_source": "ncu --set full dram__bytes_read.sum + dram__bytes_write.sum, one launch "
                          "(profiles/traffic.json)" if traffic else None,
        "peak_source": f"{peak_src} (MEASURED_PEAKS.json hbm_gbs)",
        "algorithmic_bytes_per_launch": vbytes_local,
        "launch_ms": pass_ms, "launch_samples": pass_samples,
    }
    # iteration roofline of BASELINE.md section 3: the slower of reading V once at HBM bandwidth
    # and 10 F N K flops at the tensor peak of the arithmetic the pass runs in, measured on this
    # pool's B200 with tools/tensor_peaks.cu (profiles/r02_tensor_peaks.txt)
    t_hbm = c["F"] * c["N"] * esize / world / (hbm * 1e9) * 1e3
    t_tc = 10.0 * c["F"] * c["N"] * c["K"] / world / (TENSOR_PEAK_TFLOPS[c["dtype"]] * 1e12) * 1e3
    roofline.update({
        "iteration_roofline_ms": max(t_hbm, t_tc),
        "iteration_frac": max(t_hbm, t_tc) / (ms / args.steps),
        "iteration_hbm_ms": t_hbm, "iteration_tensor_ms": t_tc,
        "iteration_bound": "hbm" if t_hbm >= t_tc else "tensor",
        "tensor_peak_tflops": TENSOR_PEAK_TFLOPS[c["dtype"]],
        "tensor_peak_source": "tools/tensor_peaks.cu on this pool's B200 "
                              "(profiles/r02_tensor_peaks.txt): tcgen05 kind::tf32 1114.4 TFLOP/s "
                              "dense / 3 for 3xTF32; mma.sync.m8n8k4.f64 37.1 TFLOP/s",
    })
    out = {
        "metric": METRIC, "value": value, "unit": "iterations/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32" if c["dtype"] == "fp32" else "f64", "data": "synthetic",
        "config": workload_config(args, world), "schedule": sched,
        "gpu_launches": launches * args.steps, "roofline": roofline,
        "clocks": clocks.summary(), "final_objective": float(obj[-1]) if done else None,
        "iterations_done": int(done),
    }
    if e2e:
        out["e2e"] = e2e
    if world == 1 and not args.no_cpu:
        dt, info = time_reference(args.config, args.algo, 1, 3)
        out["cpu_baseline"] = {
            "value": 1.0 / (dt * info["scale"]), "unit": "iterations/s", "cores": info["cores"],
            "kind": info["kind"], "sample": info["sample"]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
