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
HEADERS = ["errors", "rng", "tensor", "soft_topk", "model", "attention", "policy", "distill", "evictsim", "checkpoint"]


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


def _ref_run(cfg, tokens, budgets, select, lkv_seed, sim_seed, decode):
    """The same scenario through the reference's OWN compiled code (oracle/_ref)."""
    import ctypes as C

    import numpy as np

    import oracle as O

    R = O.ref_lib()
    L, Hq, H, d, V, maxlen, seed = cfg
    R.ref_model_create.restype = C.c_void_p
    R.ref_model_create.argtypes = [C.c_int] * 7 + [C.c_ulonglong]
    h = R.ref_model_create(L, Hq, H, d, V, maxlen, 0, seed)
    t, n = len(tokens), L * H
    I32 = lambda a: np.ascontiguousarray(a, np.int32)  # noqa: E731
    P = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    tk, bd = I32(tokens), I32(budgets)
    logits = np.empty((t, V))
    keys = np.empty((n, t, d))
    vals = np.empty((n, t, d))
    R.ref_forward_full.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
    assert R.ref_forward_full(h, P(tk), t, P(logits), P(keys), P(vals)) == 0
    rows = int(bd.sum())
    lens = np.empty(n, np.int32)
    ck, cv = np.empty((max(rows, 1), d)), np.empty((max(rows, 1), d))
    pos = np.empty(max(rows, 1), np.int32)
    rep = np.empty(4)
    R.ref_prefill_with_eviction.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_ulonglong,
                                            C.c_ulonglong] + [C.c_void_p] * 5
    assert R.ref_prefill_with_eviction(h, P(tk), t, P(bd), select, lkv_seed, sim_seed, P(lens), P(ck), P(cv), P(pos),
                                       P(rep)) == 0
    off = np.zeros(n, np.int64)
    off[1:] = np.cumsum(lens)[:-1]
    dl = np.empty((len(decode), V))
    nk = np.empty((len(decode), n, d))
    nv = np.empty((len(decode), n, d))
    ts = np.zeros(1, np.int32)
    R.ref_decode_steps.argtypes = [C.c_void_p] * 6 + [C.c_int, C.c_void_p, C.c_int] + [C.c_void_p] * 4
    assert R.ref_decode_steps(h, P(lens), P(off), P(ck), P(cv), P(pos), t, P(I32(decode)), len(decode), P(dl), P(nk),
                              P(nv), P(ts)) == 0
    R.ref_model_free.argtypes = [C.c_void_p]
    R.ref_model_free(h)
    return logits, lens, off, ck, cv, pos, rep, dl


@pytest.mark.gpu
@pytest.mark.parametrize("select", [0, 2, 3, 4])
def test_dropin_equals_reference_code(select):
    """forward_full, prefill_with_eviction (learned LKV-T selection or a baseline) and decode over the
    compacted cache through include/lkv/ on the B200 == the reference's own compiled functions
    (oracle/_ref) on the same seeded model, policy and tokens: retained positions and counts
    exact, SimReport accounting exact, fp64 values to 1e-12 (logits 1e-10 after decode)."""
    import numpy as np

    import oracle as O

    if O.ref_lib() is None:
        pytest.skip("oracle/_ref not built")
    binp = os.path.join(ROOT, "paper_2605_06676_b200", "build", "api_driver")
    if not os.path.exists(binp):
        subprocess.check_call(["make", "-s", "test_api"], cwd=os.path.join(ROOT, "paper_2605_06676_b200"))
    cfg = (2, 4, 2, 16, 96, 128, 17)
    rng = np.random.default_rng(5 + select)
    t = 57
    tokens = rng.integers(0, 96, t).tolist()
    budgets = rng.integers(0, t + 1, 4).tolist()
    budgets[1] = t
    decode = [3, 77, 12]
    args = [binp] + [str(x) for x in cfg] + ["tokens"] + [str(x) for x in tokens] + ["budgets"] + \
        [str(x) for x in budgets] + ["select", str(select), "lkv_seed", "23", "sim_seed", "9", "decode"] + \
        [str(x) for x in decode]
    r = subprocess.run(args, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    out = {}
    for line in r.stdout.splitlines():
        k, i, *v = line.split()
        out.setdefault(k, {})[i] = v
    logits, lens, off, ck, cv, pos, rep, dl = _ref_run(cfg, tokens, budgets, select, 23, 9, decode)

    def gap(a, b):
        return float(np.max(np.abs(a - b)) / (np.max(np.abs(b)) + 1e-300))

    got_logits = np.array([[float(x) for x in out["logits"][str(i)]] for i in range(t)])
    assert gap(got_logits, logits) <= 1e-12
    for i in range(4):
        v = out["head"][str(i)]
        assert int(v[0]) == lens[i] == budgets[i]
        assert [int(x) for x in v[1:]] == pos[off[i]:off[i] + lens[i]].tolist(), i
        if lens[i]:
            k = np.array([float(x) for x in out["key"][str(i)]]).reshape(-1, 16)
            assert gap(k, ck[off[i]:off[i] + lens[i]]) <= 1e-12
            vv = np.array([float(x) for x in out["val"][str(i)]]).reshape(-1, 16)
            assert gap(vv, cv[off[i]:off[i] + lens[i]]) <= 1e-12
    rline = [l for l in r.stdout.splitlines() if l.startswith("report")][0].split()[1:]
    assert int(rline[0]) == int(rep[0]) and int(rline[1]) == int(rep[1])
    assert float(rline[2]) == rep[2] and float(rline[3]) == rep[3]
    got_dl = np.array([[float(x) for x in out["dlogits"][str(s)]] for s in range(len(decode))])
    assert gap(got_dl, dl) <= 1e-10
