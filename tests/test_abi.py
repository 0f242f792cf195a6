"""CPU-side checks of the drop-in boundary: the C-ABI library loads and exports
every entry point include/lkv_b200.h declares; host-side validation raises the
reference's error taxonomy without touching a GPU."""
import ctypes as C
import os
import re
import subprocess

import pytest

import paper_2605_06676_b200 as lkv
from paper_2605_06676_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "lkv_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lkv_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_abi():
    assert set(declared_symbols()) == set(_abi.EXPORTED)


def test_library_exports_every_declared_symbol():
    L = lkv.lib()
    for name in declared_symbols():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _abi.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (lkv_[a-z_0-9]+)", out))
    assert set(declared_symbols()) <= exported


def test_library_targets_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _abi.LIB_PATH], capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_tensor_core_and_tma_instructions_present():
    sass = subprocess.run(["cuobjdump", "-sass", _abi.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass  # tcgen05.mma (scorer)
    assert "UTMALDG" in sass  # TMA tile loads
    assert "LDTM" in sass     # tcgen05.ld (TMEM epilogue)
    # the K/V projection runs on CTA pairs: tcgen05.mma.cta_group::2, 2-SM TMA, multicast commit
    assert "UTCHMMA.2CTA" in sass and "UTMALDG.2D.2CTA" in sass and "UTCBAR.2CTA.MULTICAST" in sass


def test_status_names_and_version():
    L = lkv.lib()
    assert L.lkv_abi_version() == 2
    assert L.lkv_status_name(3) == b"budget_error"
    assert L.lkv_status_name(1) == b"contract_error"


def test_host_validation_without_gpu():
    L = lkv.lib()
    lens = (C.c_int32 * 1)(100)
    # target ratio outside (0,1) -> budget_error before any device work (policy.cpp:111)
    assert L.lkv_budgets(None, 8, 1.5, 0, lens, 1, 0, None, None, None, None, 0, None) == _abi.BUDGET
    assert L.lkv_budgets(None, 8, 0.0, 0, lens, 1, 0, None, None, None, None, 0, None) == _abi.BUDGET
    # t < 1 -> contract_error (policy.cpp:123)
    zero = (C.c_int32 * 1)(0)
    assert L.lkv_budgets(C.c_void_p(16), 8, 0.5, 0, zero, 1, 0, None, C.c_void_p(16), None, C.c_void_p(256), 256,
                         None) == _abi.CONTRACT
    # malformed cache descriptor
    bad = _abi.CacheDesc(0, 1, 1, 128, 10, 1, 0, None, None, C.cast(lens, C.POINTER(C.c_int32)))
    assert L.lkv_workspace_bytes(C.byref(bad), 8) == 0
    good = _abi.CacheDesc(1, 32, 8, 128, 32768, 1, 0, None, None, C.cast((C.c_int32 * 1)(32768), C.POINTER(C.c_int32)))
    assert L.lkv_workspace_bytes(C.byref(good), 256) > 0
    cap = L.lkv_ragged_capacity(C.byref(good), 0.15, 0)
    assert cap >= 1258291


def test_error_classes_mirror_reference():
    assert issubclass(lkv.BudgetError, lkv.LkvError)
    with pytest.raises(lkv.BudgetError):
        lkv.kv_memory_bytes(retention=0.0)
    r = lkv.kv_memory_bytes(retention=1.0)
    assert r["full_bytes"] == pytest.approx(26214400000.0)  # test_evictsim.cpp:45-49
    assert abs(lkv.kv_memory_bytes(retention=0.15)["reduction_factor"] - 6.67) < 0.01


def test_host_validation_of_row4_and_comm_entry_points():
    """Host-side contract checks of the training / multi-GPU entry points (no device work)."""
    L = lkv.lib()
    # soft_topk_forward: tau must be positive (soft_topk.cpp:112), scores non-empty (:114)
    assert L.lkv_soft_topk_fwd(None, None, 0.0, 1, 8, 8, None, 0.0, None, None, None, None, None, 0, None) == _abi.CONTRACT
    assert L.lkv_soft_topk_fwd(None, None, 0.0, 1, 0, 8, None, 1.0, None, None, None, None, None, 0, None) == _abi.CONTRACT
    assert L.lkv_soft_topk_vjp(None, None, 1, 8, 8, -1.0, None, None, None) == _abi.CONTRACT
    # masked attention: empty extents / first row admits no key (attention.cpp:34,43) / GQA ratio
    a = _abi.AttnDesc(1, 4, 1, 16, 16, 128, 1, 1, -1, 0, 0.1)
    assert L.lkv_attn_workspace_bytes(C.byref(a)) == 0
    assert L.lkv_masked_attention_fwd(C.byref(a), None, None, None, None, None, None, None, 0, None) == _abi.CONTRACT
    a = _abi.AttnDesc(1, 3, 2, 16, 16, 128, 1, 1, 0, 0, 0.1)
    assert L.lkv_masked_attention_fwd(C.byref(a), None, None, None, None, None, None, None, 0, None) == _abi.CONTRACT
    a = _abi.AttnDesc(1, 4, 1, 16, 16, 64, 1, 1, 0, 0, 0.1)  # bf16 needs head_dim 128
    assert L.lkv_masked_attention_fwd(C.byref(a), None, None, None, None, None, None, None, 0, None) == _abi.UNSUPPORTED
    a = _abi.AttnDesc(2, 8, 2, 100, 300, 128, 1, 1, 0, 0, 0.1)
    assert L.lkv_attn_workspace_bytes(C.byref(a)) >= 256 + 2 * 8 * 100 * 4
    # NCCL communicator: rank outside [0, n_ranks)
    h = C.c_void_p()
    assert L.lkv_comm_init(C.byref(h), C.create_string_buffer(128), 2, 2) == _abi.CONTRACT
    assert L.lkv_comm_size(None) == 0 and L.lkv_comm_rank(None) == -1
    # head shard: the shard's heads must lie inside the global logit vector
    lens = (C.c_int32 * 1)(100)
    cd = _abi.CacheDesc(1, 4, 8, 128, 100, 1, 0, C.c_void_p(256), C.c_void_p(256), C.cast(lens, C.POINTER(C.c_int32)))
    assert L.lkv_evict_shard(C.byref(cd), None, None, 32, 8, 0.15, 1, None, None, None, None, None, 0, None) == _abi.CONTRACT
    assert L.lkv_ragged_capacity_shard(C.byref(cd), 64, 0.15, 2) > 0
