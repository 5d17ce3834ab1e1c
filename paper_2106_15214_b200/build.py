"""Build libbnmf.so in-tree for sm_100a with nvcc (no JIT cache, no torch).

    python -m paper_2106_15214_b200.build        # or build(verbose=True)

Each .cu translation unit is compiled to an object in parallel, then linked
against the NCCL shared library of the image (nvidia-nccl wheel).
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
OUT = os.environ.get("BNMF_LIB_OUT") or os.path.join(HERE, "libbnmf.so")
OBJDIR = os.path.join(HERE, "build")
SOURCES = ["engine.cu", "fused_tc.cu", "sparse.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    cands = []
    for base in {sysconfig.get_paths()["purelib"], sysconfig.get_paths()["platlib"]}:
        cands.append(os.path.join(base, "nvidia", "nccl"))
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")):
            return os.path.join(c, "include"), os.path.join(c, "lib")
    raise RuntimeError("nccl.h not found (nvidia-nccl wheel missing)")


def nvcc():
    exe = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(exe):
        raise RuntimeError("nvcc not found")
    return exe


def _deps():
    files = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    files.append(os.path.join(ROOT, "include", "bnmf.h"))
    files.append(os.path.abspath(__file__))
    return files


def up_to_date():
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(f) <= t for f in _deps())


def build(verbose=False, force=False):
    if not force and up_to_date():
        return OUT
    inc, lib = nccl_dirs()
    os.makedirs(OBJDIR, exist_ok=True)
    common = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "-Xptxas", "-v" if verbose else "-O3", f"-I{inc}", f"-I{os.path.join(ROOT, 'include')}",
              "--expt-relaxed-constexpr"]
    if os.environ.get("BNMF_WATCHDOG", "0") == "1":
        common.append("-DBNMF_WATCHDOG")
    for flag in os.environ.get("BNMF_DEFS", "").split():
        common.append(f"-D{flag}")
    if os.environ.get("BNMF_TC_PROF", "0") == "1":
        common.append("-DBNMF_TC_PROF")
    srcs = [s for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]

    def compile_one(src):
        obj = os.path.join(OBJDIR, src.replace(".cu", ".o"))
        cmd = common + ["-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        if verbose:
            sys.stderr.write(r.stderr)
        return obj

    with cf.ThreadPoolExecutor(len(srcs)) as ex:
        objs = list(ex.map(compile_one, srcs))
    tmp = OUT + ".tmp"
    cmd = [nvcc(), *ARCH, "-shared", "-o", tmp, *objs, f"-L{lib}", "-l:libnccl.so.2",
           "-Xlinker", f"-rpath,{lib}", "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force=True))
