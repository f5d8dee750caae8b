"""CPU-side checks of the C ABI (-m "not gpu"): the library builds for sm_100a, loads, and
exports every function include/uellm.h declares; struct sizes agree; pure host functions work
without a GPU."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "uellm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(uellm_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2409_14961_b200 import uellm
    return uellm


def test_exports_every_declared_symbol(lib):
    funcs = _header_functions()
    assert "uellm_profile_load" in funcs and "uellm_schedule_batches" in funcs and "uellm_batch_stats" in funcs
    out = subprocess.check_output(["nm", "-D", "--defined-only", lib.LIBRARY_PATH]).decode()
    exported = set(re.findall(r"\bT (uellm_\w+)", out))
    missing = [f for f in funcs if f not in exported]
    assert not missing, missing
    for f in funcs:
        getattr(lib._lib, f)          # resolvable through ctypes


def test_sm100a_cubin(lib):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib.LIBRARY_PATH]).decode()
    assert "sm_100a" in out


def test_host_only_calls(lib):
    assert lib._lib.uellm_abi_version() == 3
    assert lib.exchange_bytes(0) == 144 and lib.exchange_bytes(32) == 144 and lib.exchange_bytes(95) == 144
    assert lib.exchange_workspace_bytes(1000, 0) == 0 and lib.exchange_workspace_bytes(1000, 4) > 0
    assert lib.status_string(0) == "UELLM_OK" and lib.status_string(2) == "UELLM_ERR_CONTRACT"
    import workloads as W
    cfg = lib.make_config(W.SchedConfig(max_batch=256))
    a = lib.workspace_bytes(1000, cfg)
    b = lib.workspace_bytes(100000, cfg)
    assert 0 < a < b
    assert lib._lib.uellm_workspace_bytes(10, None) == 0


def test_argument_errors_without_device(lib):
    import workloads as W
    cfg = lib.make_config(W.SchedConfig())
    p = lib.Profile()
    assert lib._lib.uellm_profile_load(None, C.byref(cfg), None, 0, None, C.byref(p)) == lib.ERR_ARG
    q = lib.Queries(5, None, None, None)
    assert lib._lib.uellm_profile_load(C.byref(q), C.byref(cfg), None, 0, None, C.byref(p)) == lib.ERR_ARG
    bad = lib.make_config(W.SchedConfig(max_batch=0))
    q0 = lib.Queries(0, None, None, None)
    assert lib._lib.uellm_profile_load(C.byref(q0), C.byref(bad), None, 0, None, C.byref(p)) == lib.ERR_CONFIG
    big = lib.make_config(W.SchedConfig(max_batch=5000))
    assert lib._lib.uellm_profile_load(C.byref(q0), C.byref(big), None, 0, None, C.byref(p)) == lib.ERR_UNSUPPORTED
    # schedule on an unloaded profile
    assert lib._lib.uellm_schedule_batches(C.byref(p), C.byref(cfg), None, None, None, None) == lib.ERR_ARG
    # a9 combine: NULL / inconsistent query ranges are argument errors (checked before any device call)
    qb = (C.c_uint64 * 3)(0, 10, 5)
    assert lib._lib.uellm_exchange_combine(None, 2, 10, qb, None, 0, None, None, None, None) == lib.ERR_ARG
    assert lib._lib.uellm_exchange_pack(C.byref(p), C.byref(cfg), None, None, 0, None) == lib.ERR_ARG
    assert lib._lib.uellm_totals_combine(None, 1, 128, None, None, 0, None) == lib.ERR_ARG


def test_product_does_not_import_oracle():
    """The product path never loads the oracle (and the oracle never includes product code)."""
    pkg = os.path.join(ROOT, "paper_2409_14961_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"(import\s+oracle|from\s+oracle|liboracle|uellm_oracle|orc_)", txt), f
    orc = open(os.path.join(ROOT, "oracle", "uellm_oracle.c")).read()
    includes = re.findall(r"#include\s*[<\"]([^>\"]+)", orc)
    assert all(not i.endswith(("uellm.h", ".cuh")) for i in includes), includes
