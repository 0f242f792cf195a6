"""The reference's hot-path test expectations, ported to the C++ drop-in layer
(include/lkv_b200_dropin.hpp) and run as a native binary (tests/cpp/test_dropin.cpp)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2605_06676_b200")
BIN = os.path.join(PKG, "build", "test_dropin")


def _ensure_built():
    if not os.path.exists(BIN):
        subprocess.check_call(["make", "-s", "test_dropin"], cwd=PKG)


def test_dropin_symbols_exported():
    """Every function the C++ drop-in header declares is defined in liblkv_b200.so."""
    out = subprocess.run(["nm", "-DC", "--defined-only", os.path.join(PKG, "liblkv_b200.so")], capture_output=True,
                         text=True).stdout
    hdr = open(os.path.join(ROOT, "include", "lkv_b200_dropin.hpp")).read()
    hdr = re.sub(r"//.*", "", hdr)
    names = set(re.findall(r"^[A-Za-z].*?\b([a-z_0-9]+)\(", hdr, flags=re.M)) - {"explicit", "at", "head", "retained",
                                                                                "param_count"}
    assert {"allocate_budgets", "freeze_budgets", "token_scores", "inference_select", "hard_topk", "cache_from_trace",
            "prefill_with_eviction", "decode_attention", "kv_memory_bytes", "load_lkv_params", "head_scores"} <= names
    for n in sorted(names):
        assert re.search(r"lkv::b200::" + n + r"(\[abi:cxx11\])?\(", out), n


def test_dropin_binary_links():
    _ensure_built()
    out = subprocess.run(["ldd", BIN], capture_output=True, text=True).stdout
    assert "liblkv_b200.so" in out and "not found" not in out


@pytest.mark.gpu
def test_dropin_reference_tests_on_b200():
    _ensure_built()
    r = subprocess.run([BIN, os.path.join(ROOT, "tests", "golden")], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert re.search(r"(\d+) passed, 0 failed", r.stdout)
