"""ctypes binding of libbnmf.so (include/bnmf.h).

This is the only way the package reaches the GPU.  There is no CPU fallback:
if the library is missing or no CUDA device is visible, every solver entry
point raises ``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BNMF_LIB") or os.path.join(HERE, "libbnmf.so")

BNMF_FP64, BNMF_FP32 = 0, 1
BNMF_JMM, BNMF_BMM = 0, 1
SCHED = {"auto": 0, "reference": 1, "fused": 2}
SCHED_NAMES = {v: k for k, v in SCHED.items()}


class NativeUnavailable(RuntimeError):
    """libbnmf.so is not built or cannot run here (no CUDA device)."""


BNMF_E_ARG = -1   # include/bnmf.h


class NativeError(RuntimeError):
    """A libbnmf call returned an error code."""


class Params(C.Structure):
    _fields_ = [
        ("algorithm", C.c_int),
        ("sub_iters", C.c_int),
        ("sub_iters_w", C.c_int),
        ("sub_iters_h", C.c_int),
        ("beta", C.c_double),
        ("gamma", C.c_double),
        ("kappa", C.c_double),
        ("floor", C.c_double),
        ("tol", C.c_double),
        ("compute_kkt", C.c_int),
        ("schedule", C.c_int),
    ]


_lib = None
_lock = threading.Lock()

_SIGS = {
    "bnmf_abi_version": ([], C.c_int),
    "bnmf_device_count": ([C.POINTER(C.c_int)], C.c_int),
    "bnmf_ctx_create": ([C.POINTER(C.c_void_p), C.c_int, C.c_int], C.c_int),
    "bnmf_ctx_destroy": ([C.c_void_p], None),
    "bnmf_last_error": ([C.c_void_p], C.c_char_p),
    "bnmf_nccl_unique_id": ([C.c_void_p], C.c_int),
    "bnmf_ctx_init_comm": ([C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int64], C.c_int),
    "bnmf_set_dense": ([C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int64, C.c_int64,
                        C.c_int64, C.c_double], C.c_int),
    "bnmf_set_factors": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int], C.c_int),
    "bnmf_set_csr": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                      C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int], C.c_int),
    "bnmf_begin": ([C.c_void_p, C.POINTER(Params), C.c_int64], C.c_int),
    "bnmf_step": ([C.c_void_p, C.c_int64], C.c_int),
    "bnmf_step_timed": ([C.c_void_p, C.c_int64, C.POINTER(C.c_float)], C.c_int),
    "bnmf_sync": ([C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int)], C.c_int),
    "bnmf_read_trace": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64], C.c_int),
    "bnmf_get_factors": ([C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "bnmf_run": ([C.c_void_p, C.POINTER(Params), C.c_int64, C.POINTER(C.c_int64),
                  C.POINTER(C.c_int)], C.c_int),
    "bnmf_launches_per_iter": ([C.c_void_p, C.POINTER(C.c_int)], C.c_int),
    "bnmf_active_schedule": ([C.c_void_p, C.POINTER(C.c_int)], C.c_int),
    "bnmf_stream": ([C.c_void_p], C.c_void_p),
    "bnmf_set_profiling": ([C.c_void_p, C.c_int], C.c_int),
    "bnmf_pass_time": ([C.c_void_p, C.POINTER(C.c_float), C.POINTER(C.c_int)], C.c_int),
    "bnmf_pass_info": ([C.c_void_p, C.POINTER(C.c_int)], C.c_int),
    "bnmf_data_stats": ([C.c_void_p, C.POINTER(C.c_double)], C.c_int),
    "bnmf_kernel": ([C.c_void_p, C.c_int, C.POINTER(Params), C.c_void_p, C.c_void_p], C.c_int),
}

OP_OBJECTIVE, OP_KKT, OP_BMM_W, OP_BMM_H, OP_JMM_W, OP_JMM_H = range(6)


def load(path=LIB_PATH):
    """Load (once) and return the ctypes library; raise if it is not built."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeUnavailable(
                f"{path} is missing: build it with `python -m paper_2106_15214_b200.build`")
        lib = C.CDLL(path)
        for name, (args, res) in _SIGS.items():
            fn = getattr(lib, name, None)
            if fn is None:
                raise NativeUnavailable(f"{path} does not export {name}")
            fn.argtypes = args
            fn.restype = res
        if lib.bnmf_abi_version() != 1:
            raise NativeUnavailable("libbnmf ABI version mismatch")
        _lib = lib
        return lib


def device_count():
    lib = load()
    n = C.c_int(0)
    lib.bnmf_device_count(C.byref(n))
    return n.value


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


class Context:
    """One device context (one GPU, one stream)."""

    def __init__(self, device=0, dtype="fp64"):
        self.lib = load()
        if device_count() < 1:
            raise NativeUnavailable("no CUDA device visible to libbnmf")
        self.dtype = BNMF_FP64 if dtype in ("fp64", "float64", np.float64) else BNMF_FP32
        h = C.c_void_p()
        self._check(self.lib.bnmf_ctx_create(C.byref(h), int(device), self.dtype), None)
        self.h = h
        self.F = self.N = self.K = 0

    def _check(self, rc, h="self"):
        if rc != 0:
            handle = self.h if h == "self" else None
            msg = self.lib.bnmf_last_error(handle)
            raise NativeError(f"libbnmf error {rc}: {msg.decode() if msg else ''}")

    def close(self):
        if getattr(self, "h", None):
            self.lib.bnmf_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- setup -------------------------------------------------------------

    def init_comm(self, rank, nranks, uid, n_global):
        buf = C.create_string_buffer(bytes(uid), 128)
        self._check(self.lib.bnmf_ctx_init_comm(self.h, rank, nranks, buf, int(n_global)))

    @staticmethod
    def nccl_unique_id():
        lib = load()
        buf = C.create_string_buffer(128)
        if lib.bnmf_nccl_unique_id(buf) != 0:
            raise NativeError(lib.bnmf_last_error(None).decode())
        return buf.raw

    def set_dense(self, v, kappa=0.0):
        """v: 2-D host array (float64 or float32, C-contiguous rows) or a
        (ptr, dtype, F, N, ld) tuple describing device memory."""
        if isinstance(v, tuple):
            ptr, dt, F, N, ld = v
            src = BNMF_FP64 if dt == "fp64" else BNMF_FP32
            self._check(self.lib.bnmf_set_dense(self.h, C.c_void_p(ptr), src, 1, F, N, ld,
                                                float(kappa)))
        else:
            v = np.asarray(v)
            if v.dtype not in (np.float64, np.float32):
                v = v.astype(np.float64)
            if v.strides[1] != v.itemsize:
                v = np.ascontiguousarray(v)
            F, N = v.shape
            ld = v.strides[0] // v.itemsize
            src = BNMF_FP64 if v.dtype == np.float64 else BNMF_FP32
            self._check(self.lib.bnmf_set_dense(self.h, _ptr(v), src, 0, F, N, ld,
                                                float(kappa)))
        self.F, self.N = F, N

    def data_stats(self):
        """(min, max, sum, non-finite count, count) of the values of the last
        set_dense, before the kappa shift, computed on the device."""
        out = (C.c_double * 5)()
        self._check(self.lib.bnmf_data_stats(self.h, out))
        return tuple(out)

    def set_csr(self, indptr, indices, values, colptr, rowidx, perm, shape):
        """Host CSR (+ CSC view) of the local rows of V (see include/bnmf.h)."""
        arrs = [np.ascontiguousarray(indptr, dtype=np.int64),
                np.ascontiguousarray(indices, dtype=np.int32),
                np.ascontiguousarray(values, dtype=np.float32),
                np.ascontiguousarray(colptr, dtype=np.int64),
                np.ascontiguousarray(rowidx, dtype=np.int32),
                np.ascontiguousarray(perm, dtype=np.int32)]
        F, N = shape
        self._check(self.lib.bnmf_set_csr(self.h, *[_ptr(a) for a in arrs], int(F), int(N),
                                          int(arrs[1].size), 0))
        self.F, self.N = int(F), int(N)

    def set_factors(self, w, h):
        w = np.ascontiguousarray(w, dtype=np.float64)
        h = np.ascontiguousarray(h, dtype=np.float64)
        if w.shape[0] != self.F or h.shape[1] != self.N or w.shape[1] != h.shape[0]:
            raise ValueError("factor shapes do not match the data")
        self.K = w.shape[1]
        rc = self.lib.bnmf_set_factors(self.h, _ptr(w), _ptr(h), self.K, 0)
        if rc == BNMF_E_ARG:
            # the FactorPair checks, made on the device copy (core.py: FactorPair.__post_init__)
            msg = self.lib.bnmf_last_error(self.h)
            msg = msg.decode() if msg else ""
            if msg.startswith("factor entries"):
                raise ValueError(msg)
        self._check(rc)

    # -- running -----------------------------------------------------------

    def begin(self, params, max_iters):
        self._params = params
        self._check(self.lib.bnmf_begin(self.h, C.byref(params), int(max_iters)))

    def step(self, n):
        self._check(self.lib.bnmf_step(self.h, int(n)))

    def step_timed(self, n):
        ms = C.c_float(0.0)
        self._check(self.lib.bnmf_step_timed(self.h, int(n), C.byref(ms)))
        return ms.value

    def sync(self):
        done = C.c_int64(0)
        conv = C.c_int(0)
        self._check(self.lib.bnmf_sync(self.h, C.byref(done), C.byref(conv)))
        return done.value, bool(conv.value)

    def run(self, params, max_iters):
        done = C.c_int64(0)
        conv = C.c_int(0)
        self._check(self.lib.bnmf_run(self.h, C.byref(params), int(max_iters),
                                      C.byref(done), C.byref(conv)))
        return done.value, bool(conv.value)

    def trace(self, n):
        obj = np.empty(n)
        sec = np.empty(n)
        kkt = np.empty((n, 2))
        if n:
            self._check(self.lib.bnmf_read_trace(self.h, _ptr(obj), _ptr(sec), _ptr(kkt), n))
        return obj, sec, kkt

    def factors(self):
        w = np.empty((self.F, self.K))
        h = np.empty((self.K, self.N))
        self._check(self.lib.bnmf_get_factors(self.h, _ptr(w), _ptr(h)))
        return w, h

    def kernel(self, op, params, cur=None):
        """One kernel of the reference's lower-level API (include/bnmf.h: bnmf_kernel) on the
        data and factor pair this context holds; returns a float (objective), a pair (KKT) or
        the updated factor."""
        if op in (OP_BMM_W, OP_JMM_W):
            out = np.empty((self.F, self.K))
        elif op in (OP_BMM_H, OP_JMM_H):
            out = np.empty((self.K, self.N))
        else:
            out = np.empty(2)
        if cur is not None:
            cur = np.ascontiguousarray(cur, dtype=np.float64)
            want = (self.K, self.N) if op == OP_JMM_W else (self.F, self.K)
            if cur.shape != want:
                raise ValueError(f"current factor has shape {cur.shape}, expected {want}")
        self._check(self.lib.bnmf_kernel(self.h, int(op), C.byref(params),
                                         _ptr(cur) if cur is not None else None, _ptr(out)))
        if op == OP_OBJECTIVE:
            return float(out[0])
        if op == OP_KKT:
            return float(out[0]), float(out[1])
        return out

    def launches_per_iter(self):
        n = C.c_int(0)
        self._check(self.lib.bnmf_launches_per_iter(self.h, C.byref(n)))
        return n.value

    def set_profiling(self, on=True):
        self._check(self.lib.bnmf_set_profiling(self.h, 1 if on else 0))

    def pass_time(self):
        ms = C.c_float(0.0)
        n = C.c_int(0)
        self._check(self.lib.bnmf_pass_time(self.h, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def pass_info(self):
        """(kernel, grid CTAs, CTAs per cluster, rows of cluster rank 0) of the fused pass
        the last begin() selected; kernel is "none", "simt" or "tcgen05"."""
        out = (C.c_int * 4)()
        self._check(self.lib.bnmf_pass_info(self.h, out))
        return {0: "none", 1: "simt", 2: "tcgen05"}[out[0]], out[1], out[2], out[3]

    def schedule(self):
        n = C.c_int(0)
        self._check(self.lib.bnmf_active_schedule(self.h, C.byref(n)))
        return SCHED_NAMES.get(n.value, str(n.value))
