"""CPU-side checks of the C ABI: the library builds, loads and exports every
symbol include/bnmf.h declares.  No compute calls (no GPU here)."""

import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "bnmf.h")


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(bnmf_[a-z_0-9]+)\s*\(", txt)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ("bnmf_ctx_create", "bnmf_set_dense", "bnmf_set_factors", "bnmf_begin",
              "bnmf_step", "bnmf_sync", "bnmf_read_trace", "bnmf_get_factors", "bnmf_run"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2106_15214_b200 import build
    path = build.build()
    import ctypes
    lib = ctypes.CDLL(path)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.bnmf_abi_version() == 1


def test_native_loader_is_strict_without_gpu():
    from paper_2106_15214_b200 import _native
    _native.load()
    if _native.device_count() == 0:
        with pytest.raises(_native.NativeUnavailable):
            _native.Context(0, "fp64")


def test_sm100a_cubin_embedded():
    import subprocess
    from paper_2106_15214_b200 import build
    path = build.build()
    out = subprocess.run(["cuobjdump", "-lelf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out
