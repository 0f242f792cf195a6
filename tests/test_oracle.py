"""Pins the CPU oracle (oracle/) against the reference's own known answers.

Each case restates a test of the reference suite for this path (file:line under
/root/reference/proj/tests) and, where the reference's own soft_topk.cpp /
policy.cpp were compiled into oracle/_ref, checks the restatement bit-for-bit
against them on seeded random instances.  CPU only.
"""
import math

import numpy as np
import pytest

import oracle as O


# ---- soft_topk (test_soft_topk.cpp) -------------------------------------------
def test_laplace_cdf_anchor_points():  # test_soft_topk.cpp:26-34
    assert O.laplace_cdf(0.0) == pytest.approx(0.5, rel=1e-15)
    assert O.laplace_cdf(math.log(2.0)) == pytest.approx(0.75, rel=1e-15)
    assert O.laplace_cdf(-math.log(2.0)) == pytest.approx(0.25, rel=1e-15)
    for z in (0.3, 1.7, 9.0):
        assert O.laplace_cdf(-z) == pytest.approx(1.0 - O.laplace_cdf(z), rel=1e-14)


def test_threshold_all_equal_quarter_budget():  # test_soft_topk.cpp:36-41
    lam, m = O.solve_threshold([0.0, 0.0, 0.0, 0.0], 1.0)
    assert lam == pytest.approx(math.log(2.0), rel=1e-12)
    assert m == 0


def test_golden_threshold_2_1_0():  # test_soft_topk.cpp:43-50
    x = [2.0, 1.0, 0.0]
    bis = O.bisect_lambda(x, 1.5)
    assert bis == pytest.approx(1.0, rel=1e-11)
    lam, _ = O.solve_threshold(x, 1.5)
    assert abs(lam - bis) < 1e-9


def test_translation_covariance():  # test_soft_topk.cpp:52-61
    x = O.random_scores(9, 77)
    l0, _ = O.solve_threshold(x, 3.3)
    for c in (-17.0, 0.25, 40.0):
        l1, _ = O.solve_threshold(x + c, 3.3)
        assert abs(l1 - (l0 + c)) < 1e-9


def test_budget_domain_errors():  # test_soft_topk.cpp:63-71
    x = O.random_scores(5, 3)
    for k in (0.0, 5.0, -1.0):
        with pytest.raises(O.OracleError) as e:
            O.solve_threshold(x, k)
        assert e.value.code == O.BUDGET
    with pytest.raises(O.OracleError) as e:
        O.soft_topk_forward(x, 6.0, 1.0)
    assert e.value.code == O.BUDGET
    for tau in (0.0, -2.0):
        with pytest.raises(O.OracleError) as e:
            O.soft_topk_forward(x, 1.0, tau)
        assert e.value.code == O.CONTRACT


def test_symmetric_forward_and_hard_limit():  # test_soft_topk.cpp:73-83
    out = O.soft_topk_forward([0.0] * 4, 1.0, 1.0)
    assert np.allclose(out["values"], 0.25, rtol=1e-12, atol=0)
    hard = O.soft_topk_forward([3.0, 1.0, 2.0], 1.0, 1e-4)["values"]
    assert abs(hard[0] - 1.0) < 1e-6 and abs(hard[1]) < 1e-6 and abs(hard[2]) < 1e-6


def test_random_instances_against_bisection():  # test_soft_topk.cpp:85-114
    meta = O.Rng(2024)
    for rep in range(60):
        n = 2 + meta.uniform_int(0, 511)
        k = meta.uniform(0.05, n - 0.05)
        tau = [0.01, 0.1, 1.0][meta.uniform_int(0, 3)]
        x = O.random_scores(n, 9000 + rep)
        out = O.soft_topk_forward(x, k, tau)
        v = out["values"]
        assert (v > 0).all() and (v < 1).all()
        assert abs(v.sum() - out["clamped_k"]) <= 1e-9 * n
        assert abs(out["threshold_lambda"] - O.bisect_lambda(x / tau, out["clamped_k"])) <= 1e-9
        order = np.argsort(-x, kind="stable")
        assert (np.diff(v[order]) <= 0).all()


def test_output_translation_invariance():  # test_soft_topk.cpp:116-127
    x = O.random_scores(32, 404)
    base = O.soft_topk_forward(x, 7.5, 1.0)["values"]
    for c in (-50.0, -1.0, 0.5, 50.0):
        moved = O.soft_topk_forward(x + c, 7.5, 1.0)["values"]
        assert np.max(np.abs(moved - base)) <= 1e-9


def test_degenerate_single_score():  # test_soft_topk.cpp:176-184
    out = O.soft_topk_forward([1.3], 0.4, 1.0)
    assert out["values"][0] == pytest.approx(0.4)


def test_hard_topk_ranking_boundaries_ties():  # test_soft_topk.cpp:190-199
    x = [0.1, 0.9, 0.5]
    assert O.hard_topk(x, 2).tolist() == [0, 1, 1]
    assert O.hard_topk(x, 0).tolist() == [0, 0, 0]
    assert O.hard_topk(x, 3).tolist() == [1, 1, 1]
    assert O.hard_topk([0.7, 0.2, 0.7], 1).tolist() == [1, 0, 0]
    for b in (4, -1):
        with pytest.raises(O.OracleError) as e:
            O.hard_topk(x, b)
        assert e.value.code == O.BUDGET


def test_hard_topk_is_stable_sort():
    rng = np.random.default_rng(5)
    for n in (1, 2, 7, 100, 1000):
        x = rng.integers(0, 5, n).astype(np.float64)  # heavy ties
        for b in (0, 1, n // 2, n):
            order = np.argsort(-x, kind="stable")
            want = np.zeros(n, np.int32)
            want[order[:b]] = 1
            assert (O.hard_topk(x, b) == want).all()
            assert (O.select_positions_f32(x.astype(np.float32), b) == np.sort(order[:b])).all()


def test_signed_zero_ties_keep_lowest_index():
    x = np.array([-0.0, 0.0, -0.0, 0.0], np.float32)
    assert O.select_positions_f32(x, 2).tolist() == [0, 1]


# ---- budgets (test_policy.cpp) ---------------------------------------------------
def test_equal_scores_allocate_target_ratio():  # test_policy.cpp:51-60
    r = O.allocate_budgets(np.full(8, 0.3), 0.15)
    assert np.allclose(r, 0.15, rtol=1e-12, atol=0)
    assert r.sum() == pytest.approx(1.2, rel=1e-12)


def test_dominant_head_gets_greatest_ratio():  # test_policy.cpp:62-68
    r = O.allocate_budgets([0, 0, 5.0, 0, 0, 0, 0, 0], 0.15)
    assert all(r[2] > r[i] for i in range(8) if i != 2)


def test_allocation_matches_bisection():  # test_policy.cpp:70-94
    rng = O.Rng(515)
    for rep in range(30):
        L = 1 + rng.uniform_int(0, 6)
        H = 1 + rng.uniform_int(0, 4)
        n = L * H
        if n < 2:
            continue
        R = rng.uniform(0.05, 0.95)
        s = np.array([rng.uniform(-2.0, 2.0) for _ in range(n)])
        r = O.allocate_budgets(s, R)
        assert ((r > 0) & (r < 1)).all()
        assert abs(r.sum() - R * n) <= 1e-9 * n
        lam = O.bisect_lambda(s, R * n)
        want = np.array([O.laplace_cdf(v - lam) for v in s])
        assert np.allclose(r, want, rtol=1e-8, atol=0)


def test_allocation_shift_invariance():  # test_policy.cpp:96-105
    rng = O.Rng(99)
    s = np.array([rng.uniform(-1.0, 1.0) for _ in range(8)])
    a = O.allocate_budgets(s, 0.2)
    b = O.allocate_budgets(s + 13.5, 0.2)
    assert np.max(np.abs(a - b)) <= 1e-9


def test_ratio_domain():  # policy.cpp:111
    for R in (0.0, 1.0, -0.1, 1.5):
        with pytest.raises(O.OracleError) as e:
            O.allocate_budgets(np.zeros(4), R)
        assert e.value.code == O.BUDGET


def test_floor_fixture():  # test_policy.cpp:107-116
    r = [0.15, 0.15, 0.003]
    assert O.freeze_budgets(r, 1000).tolist() == [150, 150, 3]
    assert O.freeze_budgets(r, 200000).tolist() == [30000, 30000, 600]
    assert O.freeze_budgets(r, 100).tolist() == [15, 15, 0]
    with pytest.raises(O.OracleError) as e:
        O.freeze_budgets(r, 0)
    assert e.value.code == O.CONTRACT


@pytest.mark.parametrize("n,t,R,sigma", [(8, 4096, 0.15, 1.0), (256, 32768, 0.15, 1.0),
                                         (256, 131072, 0.05, 1.0), (256, 131072, 0.25, 1.0),
                                         (640, 65536, 0.10, 1.5), (3, 1000, 0.4, 0.3)])
def test_exact_sum_budgets(n, t, R, sigma):
    rng = np.random.default_rng(n + t)
    logits = rng.normal(0, sigma, n)
    r = O.allocate_budgets(logits, R)
    b = O.freeze_budgets_exact(r, R, t)
    fl = O.freeze_budgets(r, t)
    assert int(b.sum()) == round(R * n * t)
    assert ((b - fl >= 0) & (b - fl <= 1)).all()
    assert ((b >= 0) & (b <= t)).all()
    # the +1s go to the largest remainders (ties to the lower index)
    rem = r * t - np.floor(r * t)
    got = np.nonzero(b - fl)[0]
    order = sorted(range(n), key=lambda i: (-rem[i], i))
    assert sorted(got.tolist()) == sorted(order[: len(got)])


def test_config_totals():  # exact totals per BASELINE config
    for n, t, R, want in [(8, 4096, 0.15, 4915), (256, 32768, 0.15, 1258291), (256, 131072, 0.05, 1677722),
                          (256, 131072, 0.10, 3355443), (256, 131072, 0.15, 5033165),
                          (256, 131072, 0.25, 8388608), (640, 65536, 0.10, 4194304)]:
        assert round(R * n * t) == want


def test_token_scorer_pointwise_and_zero_preserving():  # test_policy.cpp:118-139
    rng = np.random.default_rng(13)
    t, d, hid = 6, 16, 16
    k = rng.uniform(-1, 1, (t, d)).astype(np.float32)
    v = rng.uniform(-1, 1, (t, d)).astype(np.float32)
    k[4], v[4] = k[2], v[2]
    w1 = rng.normal(0, 1 / math.sqrt(2 * d), (2 * d, hid))
    w2 = rng.normal(0, 1 / math.sqrt(hid), hid)
    u = O.token_scores(k, v, w1, np.zeros(hid), w2, act=O.SILU)
    assert u[2] == u[4]
    uz = O.token_scores(np.zeros((t, d), np.float32), np.zeros((t, d), np.float32), w1, np.zeros(hid), w2)
    assert (uz == 0.0).all()


def test_token_scorer_formula():
    rng = np.random.default_rng(3)
    t, d, hid = 9, 8, 4
    k = rng.normal(size=(t, d)).astype(np.float32)
    w1 = rng.normal(size=(d, hid))
    b1 = rng.normal(size=hid)
    w2 = rng.normal(size=hid)
    h = k.astype(np.float64) @ w1 + b1
    from math import erf
    gelu = np.vectorize(lambda x: 0.5 * x * (1 + erf(x / math.sqrt(2))))(h)
    assert np.allclose(O.token_scores(k, None, w1, b1, w2, act=O.GELU_ERF), gelu @ w2, rtol=1e-12, atol=1e-12)
    silu = h / (1 + np.exp(-h))
    v = rng.normal(size=(t, d)).astype(np.float32)
    w1kv = rng.normal(size=(2 * d, hid))
    hk = np.concatenate([k, v], 1).astype(np.float64) @ w1kv + b1
    assert np.allclose(O.token_scores(k, v, w1kv, b1, w2, act=O.SILU), (hk / (1 + np.exp(-hk))) @ w2,
                       rtol=1e-12, atol=1e-12)


# ---- memory model (test_evictsim.cpp:45-80) ---------------------------------------
def test_kv_storage_fixtures():
    full = O.kv_memory_bytes(retention=1.0)
    assert full["full_bytes"] == pytest.approx(26214400000.0)
    r15 = O.kv_memory_bytes(retention=0.15)
    assert r15["reduction_factor"] == pytest.approx(1 / 0.15, rel=1e-12)
    assert abs(r15["reduction_factor"] - 6.67) < 0.01
    prev = 0.0
    for r in (0.1, 0.2, 0.5, 0.8, 1.0):
        c = O.kv_memory_bytes(retention=r)["compressed_bytes"]
        assert c > prev
        prev = c
    for r in (0.0, 1.5):
        with pytest.raises(O.OracleError):
            O.kv_memory_bytes(retention=r)
    rep = O.kv_memory_bytes(1, 2, 4, 2.0, 100, budgets=[15, 14])
    assert rep["full_bytes"] == pytest.approx(2 * 4 * 2.0 * 2 * 100)
    assert rep["compressed_bytes"] == pytest.approx((15 + 14) * 4 * 2.0 * 2)


# ---- decode attention (test_attention.cpp, oracles.hpp:44-75) ----------------------
def _logspace_attention(q, k, v, scale):
    s = scale * (q @ k.T)
    s = s - s.max(axis=1, keepdims=True)
    p = np.exp(s)
    p /= p.sum(axis=1, keepdims=True)
    return p @ v


@pytest.mark.parametrize("t", [1, 2, 9, 257])
def test_decode_attention_matches_logspace(t):  # test_attention.cpp:63-71
    rng = np.random.default_rng(t)
    G, d = 4, 8
    q = rng.normal(size=(G, d))
    k = rng.normal(size=(t, d)).astype(np.float32)
    v = rng.normal(size=(t, d)).astype(np.float32)
    out = O.decode_attention(q, k, v, 1 / math.sqrt(d))
    assert np.max(np.abs(out - _logspace_attention(q, k.astype(np.float64), v.astype(np.float64),
                                                   1 / math.sqrt(d)))) < 1e-10
    if t == 1:  # single key renormalises to the value row (test_attention.cpp:55-61)
        assert np.allclose(out, v.astype(np.float64)[0], rtol=1e-14)


def test_decode_attention_empty_rejected():  # attention.cpp:33
    with pytest.raises(O.OracleError) as e:
        O.decode_attention(np.zeros((1, 4)), np.zeros((0, 4), np.float32), np.zeros((0, 4), np.float32), 0.5)
    assert e.value.code == O.CONTRACT


# ---- rng ---------------------------------------------------------------------------
def test_mt19937_64_known_answer():
    # The C++ standard pins the 10000th output of a default-seeded mt19937_64.
    r = O.Rng(5489)
    for _ in range(9999):
        r.next_u64()
    assert r.next_u64() == 9981545732273789042


# ---- bit-for-bit against the reference's own code (oracle/_ref) --------------------
ref = O.ref_lib()
needs_ref = pytest.mark.skipif(ref is None, reason="oracle/_ref not built (reference sources absent)")


@needs_ref
def test_bitexact_vs_reference_solve_and_budgets():
    import ctypes as C

    rng = np.random.default_rng(11)
    for rep in range(300):
        n = int(rng.integers(2, 700))
        sigma = float(rng.choice([0.1, 1.0, 1.5, 5.0]))
        x = rng.normal(0, sigma, n)
        if rep % 7 == 0:
            x = np.round(x, 1)  # ties
        R = float(rng.uniform(0.01, 0.99))
        ratios_ref = np.empty(n)
        rc = ref.ref_allocate_budgets(x.ctypes.data_as(O._dp), 1, n, R, ratios_ref.ctypes.data_as(O._dp))
        try:
            ratios = O.allocate_budgets(x, R)
            mine = 0
        except O.OracleError as e:
            mine = e.code
        assert rc == mine
        if rc:
            continue
        assert (ratios == ratios_ref).all(), rep  # bit-exact
        for t in (1, 100, 4096, 32768, 131072):
            b_ref = np.empty(n, np.int32)
            assert ref.ref_freeze_budgets(ratios_ref.ctypes.data_as(O._dp), 1, n, t,
                                          b_ref.ctypes.data_as(O._ip)) == 0
            assert (O.freeze_budgets(ratios, t) == b_ref).all()
        lam_r, m_r = C.c_double(), C.c_int()
        assert ref.ref_solve_threshold(x.ctypes.data_as(O._dp), n, R * n, C.byref(lam_r), C.byref(m_r)) == 0
        lam, m = O.solve_threshold(x, R * n)
        assert lam == lam_r.value and m == m_r.value


@needs_ref
def test_bitexact_vs_reference_hard_topk():
    rng = np.random.default_rng(12)
    for rep in range(200):
        n = int(rng.integers(1, 3000))
        x = rng.normal(size=n)
        if rep % 2:
            x = np.round(x * 3) / 3  # many ties
        if rep % 5 == 0:
            x[rng.integers(0, n, max(1, n // 10))] = -0.0
        b = int(rng.integers(0, n + 1))
        m_ref = np.empty(n, np.int32)
        assert ref.ref_hard_topk(x.ctypes.data_as(O._dp), n, b, m_ref.ctypes.data_as(O._ip)) == 0
        assert (O.hard_topk(x, b) == m_ref).all()
    x = np.zeros(3)
    assert ref.ref_hard_topk(x.ctypes.data_as(O._dp), 3, 4, np.empty(3, np.int32).ctypes.data_as(O._ip)) == 3


@needs_ref
def test_reference_mode_scorer_vs_reference():
    rng = np.random.default_rng(14)
    t, d, hid = 37, 16, 16
    k = rng.uniform(-1, 1, (t, d))
    v = rng.uniform(-1, 1, (t, d))
    w1 = rng.normal(0, 0.2, (2 * d, hid))
    b1 = rng.normal(0, 0.1, hid)
    w2 = rng.normal(0, 0.25, hid)
    out_ref = np.empty(t)
    assert ref.ref_token_scores(k.ctypes.data_as(O._dp), v.ctypes.data_as(O._dp), t, d, w1.ctypes.data_as(O._dp),
                                b1.ctypes.data_as(O._dp), w2.ctypes.data_as(O._dp), hid,
                                out_ref.ctypes.data_as(O._dp)) == 0
    # the oracle widens float32 inputs; feed exactly representable values
    k32, v32 = k.astype(np.float32), v.astype(np.float32)
    out_ref2 = np.empty(t)
    k64, v64 = k32.astype(np.float64), v32.astype(np.float64)
    ref.ref_token_scores(k64.ctypes.data_as(O._dp), v64.ctypes.data_as(O._dp), t, d, w1.ctypes.data_as(O._dp),
                         b1.ctypes.data_as(O._dp), w2.ctypes.data_as(O._dp), hid, out_ref2.ctypes.data_as(O._dp))
    mine = O.token_scores(k32, v32, w1, b1, w2, act=O.SILU)
    assert np.max(np.abs(mine - out_ref2)) <= 1e-13 * max(1.0, np.max(np.abs(out_ref2)))


# ---------------------------------------------------------------------------------------------
# toy GQA model decode step: numpy restatement vs the reference's model.cpp
# ---------------------------------------------------------------------------------------------
from oracle import model as OM  # noqa: E402


def _trace_cache(cfg, K, V, rng, keep=0.6):
    heads = []
    t = K.shape[1]
    for i in range(cfg.total_kv_heads):
        m = rng.random(t) < keep
        idx = np.nonzero(m)[0]
        heads.append(OM.HeadCache(K[i][idx].copy(), V[i][idx].copy(), idx.astype(np.int32)))
    return heads


@needs_ref
def test_model_oracle_matches_reference_model_cpp():
    cfg = OM.ModelConfig(n_layers=3, n_query_heads=8, n_kv_heads=2, head_dim=16, vocab_size=97, max_seq_len=64)
    R = OM.RefModel(cfg)
    P = R.params()                                   # the reference's own init_model weights
    P["layers.1.attn_norm"] = 1.0 + 0.1 * np.random.default_rng(3).standard_normal(cfg.d_model)
    R.set_params(P)
    toks = np.random.default_rng(4).integers(0, cfg.vocab_size, 20)
    lr, kr, vr = R.forward_full(toks)
    lo, ko, vo = OM.forward_full(cfg, P, toks)
    assert np.abs(lo - lr).max() <= 1e-12 * np.abs(lr).max()
    assert np.abs(ko - kr).max() <= 1e-12 and np.abs(vo - vr).max() <= 1e-12
    heads = _trace_cache(cfg, kr, vr, np.random.default_rng(5))
    steps = [7, 0, 96]
    lref, nk, nv, ts = R.decode_steps(heads, 20, steps)
    mine = [OM.HeadCache(h.keys.copy(), h.values.copy(), h.positions.copy()) for h in heads]
    seen = 20
    for s, tok in enumerate(steps):
        lg, seen = OM.decode_step(cfg, P, mine, seen, tok)
        assert np.abs(lg - lref[s]).max() <= 1e-12 * np.abs(lref[s]).max(), s
        for i, hc in enumerate(mine):
            assert np.abs(hc.keys[-1] - nk[s, i]).max() <= 1e-12 and np.abs(hc.values[-1] - nv[s, i]).max() <= 1e-12
            assert hc.positions[-1] == 20 + s
    assert seen == ts == 23


def test_model_oracle_prefill_then_decode_equals_one_shot():
    """test_model.cpp:101-115: decoding token t over the full prefix cache reproduces the full
    forward's last row (<= 1e-10)."""
    cfg = OM.ModelConfig(n_layers=2, n_query_heads=4, n_kv_heads=2, head_dim=8, vocab_size=50, max_seq_len=32)
    P = OM.random_params(cfg, 11, gain=0.2)
    toks = np.random.default_rng(12).integers(0, cfg.vocab_size, 12)
    full, _, _ = OM.forward_full(cfg, P, toks)
    _, K, V = OM.forward_full(cfg, P, toks[:-1])
    heads = [OM.HeadCache(K[i].copy(), V[i].copy(), np.arange(11, dtype=np.int32)) for i in range(cfg.total_kv_heads)]
    lg, seen = OM.decode_step(cfg, P, heads, 11, int(toks[-1]))
    assert seen == 12 and np.abs(lg - full[-1]).max() <= 1e-10
