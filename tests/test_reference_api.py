"""The declaration-compatible reference API (include/lkv/*.hpp) -- the drop-in boundary.

The reference's OWN test cases for the inference path -- test_soft_topk, test_policy,
test_evictsim, test_model and test_attention, compiled unmodified from /root/reference (line
ranges chosen by oracle/Makefile `ref_tests`, nothing copied) against our headers instead of
proj/include, linked to liblkv_b200.so -- run on the B200.  A reference caller therefore switches
by changing its include path and link line only.

CPU tests: the headers compile on their own, every function they declare is exported by the
library, the test binaries exist and link.  GPU tests: the binaries pass.
"""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
INC = os.path.join(ROOT, "include")
LIB = os.path.join(ROOT, "paper_2605_06676_b200", "liblkv_b200.so")
REF_BIN = os.path.join(ROOT, "oracle", "_ref")
SUITES = ["soft_topk", "policy", "evictsim", "model", "attention"]
HEADERS = ["errors", "rng", "tensor", "soft_topk", "model", "attention", "policy", "distill", "evictsim"]


def _bin(s):
    return os.path.join(REF_BIN, f"ref_test_{s}")


def _ensure_built():
    if os.path.isdir("/root/reference/proj/tests") and not all(os.path.exists(_bin(s)) for s in SUITES):
        subprocess.check_call(["make", "-s", "ref_tests"], cwd=os.path.join(ROOT, "oracle"))


def test_headers_compile_standalone(tmp_path):
    for h in HEADERS:
        src = tmp_path / f"{h}.cpp"
        src.write_text(f'#include "lkv/{h}.hpp"\nint main() {{ return 0; }}\n')
        r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Werror", f"-I{INC}", str(src)],
                           capture_output=True, text=True)
        assert r.returncode == 0, (h, r.stderr)


def test_every_declared_function_is_exported():
    out = subprocess.run(["nm", "-DC", "--defined-only", LIB], capture_output=True, text=True).stdout
    want = {"allocate_budgets", "freeze_budgets", "token_scores", "inference_select", "hard_topk", "solve_threshold",
            "soft_topk_forward", "soft_topk_vjp", "laplace_cdf", "sample_gumbel", "cache_from_trace", "decode_step",
            "forward_full", "forward_masked", "init_model", "make_cache", "prefill_with_eviction", "kv_memory_bytes",
            "policy_budget_table", "masked_attention_dense", "masked_attention_blocked", "validate_call",
            "init_lkv_params", "head_scores", "baseline_budget", "baseline_select", "param_count",
            "budget_table_csv", "budget_kind_from_string", "select_kind_from_string", "reshape", "grad_enabled"}
    for n in sorted(want):
        assert re.search(r"\blkv::" + n + r"(\[abi:cxx11\])?\(", out), n
    for m in ["Tensor::Tensor(", "Tensor::numel(", "Tensor::from(", "Tensor::full(", "Tensor::scalar(",
              "Tensor::value(", "Tensor::detached_clone(", "ModelConfig::validate(", "MemoryModel::validate(",
              "LkvParams::named_params", "ModelWeights::named_params"]:
        assert "lkv::" + m in out, m


def test_reference_test_binaries_link():
    _ensure_built()
    for s in SUITES:
        if not os.path.exists(_bin(s)):
            pytest.skip("oracle/_ref/ref_test_* not built (needs /root/reference at build time)")
        out = subprocess.run(["ldd", _bin(s)], capture_output=True, text=True).stdout
        assert "liblkv_b200.so" in out and "not found" not in out, s
        # they were compiled against include/lkv, never against the reference's own headers
        assert "liblkv_ref" not in out


@pytest.mark.gpu
@pytest.mark.parametrize("suite", SUITES)
def test_reference_test_cases_pass_on_b200(suite):
    _ensure_built()
    if not os.path.exists(_bin(suite)):
        pytest.skip("oracle/_ref/ref_test_* not built (needs /root/reference at build time)")
    r = subprocess.run([_bin(suite)], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| 0 failed", r.stdout)
    assert m and int(m.group(1)) > 0


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["desk", "l2h4d128"])
def test_checkpoint_api_ingests_reference_policy(name, tmp_path):
    """lkv::load_lkv_params on a checkpoint written by the reference's own save path, LKV-H logits
    by lkv::head_scores on the B200 == the reference's head_scores; save/load round trips; the
    device budgets from them == the CPU oracle's freeze of the reference's logits."""
    import numpy as np

    import oracle as O

    binp = os.path.join(ROOT, "paper_2605_06676_b200", "build", "test_checkpoint_api")
    if not os.path.exists(binp):
        subprocess.check_call(["make", "-s", "test_api"], cwd=os.path.join(ROOT, "paper_2605_06676_b200"))
    g = os.path.join(ROOT, "tests", "golden")
    r = subprocess.run([binp, os.path.join(g, f"lkv_params_{name}.bin"), str(tmp_path)], capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    got = np.array([float(l.split()[2]) for l in r.stdout.splitlines() if l.startswith("score ")])
    want = np.load(os.path.join(g, f"head_scores_{name}.npy"))
    assert got.shape == want.shape
    assert np.max(np.abs(got - want)) <= 1e-12 * max(1.0, np.max(np.abs(want)))
    b = np.array([int(l.split()[2]) for l in r.stdout.splitlines() if l.startswith("budget ")])
    assert (b == O.freeze_budgets(O.allocate_budgets(want, 0.15), 1000)).all()
