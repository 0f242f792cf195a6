"""GPU parity: every stage of the CUDA path against the CPU oracle on identical inputs.

Stage-wise protocol:
  * budgets     bit-exact vs the oracle from identical logits;
  * scores      max|d| / max|ref| <= 1e-5 (fp32) or 1e-2 (bf16) vs the fp64 oracle
                on the same (bf16-rounded) inputs and weights;
  * indices     bit-exact vs the oracle's hard_topk fed the DEVICE scores;
  * layout      bit-exact rows/positions/offsets vs the oracle compaction;
  * decode      1e-5 (fp32) / 1e-2 (bf16) vs the fp64 oracle reading the device's cache.
All calls go through the C ABI (liblkv_b200.so).
"""
import math

import numpy as np
import pytest
import torch

import oracle as O
import paper_2605_06676_b200 as lkv
from paper_2605_06676_b200 import synth

pytestmark = pytest.mark.gpu
DEV = "cuda"


def rel_gap(a, b):  # gradcheck.cpp:74-81 convention
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / (np.max(np.abs(b)) + 1e-12)) if a.size else 0.0


def to_np(t: torch.Tensor):
    """Host copy in the oracle's input format (bf16 -> uint16 bit patterns)."""
    t = t.detach().contiguous().cpu()
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().view(np.uint16)
    return t.numpy()


def w_np(t: torch.Tensor):
    return t.detach().to(torch.float64).cpu().numpy()


# ---------------------------------------------------------------------------------------------
# K2 budgets
# ---------------------------------------------------------------------------------------------
def test_library_is_sm100():
    assert lkv.lib().lkv_device_check() == 0, lkv.lib().lkv_last_error()


@pytest.mark.parametrize("n,sigma", [(8, 1.0), (256, 1.0), (640, 1.5), (2, 0.3), (1, 1.0), (1000, 3.0)])
def test_budgets_bitexact(n, sigma):
    rng = np.random.default_rng(n * 7 + int(sigma * 10))
    mismatched_ratios = 0
    for rep in range(40):
        logits = rng.normal(0, sigma, n)
        if rep % 9 == 0:
            logits = np.round(logits, 1)
        R = float(rng.choice([0.05, 0.10, 0.15, 0.25, rng.uniform(0.01, 0.99)]))
        ts = [int(x) for x in rng.choice([1, 100, 4096, 8192, 32768, 65536, 131072], size=3)]
        want_r = O.allocate_budgets(logits, R)
        for mode in (lkv.BUDGET_FLOOR, lkv.BUDGET_EXACT):
            r, b = lkv.budgets(torch.tensor(logits, device=DEV), R, ts, mode)
            r = r.cpu().numpy()
            assert np.max(np.abs(r - want_r) / want_r) <= 1e-13
            mismatched_ratios += int((r != want_r).sum())
            for i, t in enumerate(ts):
                want_b = (O.freeze_budgets(want_r, t) if mode == lkv.BUDGET_FLOOR
                          else O.freeze_budgets_exact(want_r, R, t))
                assert (b[i].cpu().numpy() == want_b).all(), (rep, t, mode)
                if mode == lkv.BUDGET_EXACT:
                    assert int(b[i].sum()) == math.floor(R * n * t + 0.5)  # llround: half away from zero
    print(f"ratio elements differing in the last bits: {mismatched_ratios}")


def test_budget_fixtures():
    r = lkv.allocate_budgets(torch.full((8,), 0.3, dtype=torch.float64, device=DEV), 0.15, 4, 2)  # test_policy.cpp:51-60
    assert torch.allclose(r, torch.full_like(r, 0.15), rtol=1e-12, atol=0)
    r = lkv.allocate_budgets(torch.tensor([0, 0, 5.0, 0, 0, 0, 0, 0], device=DEV), 0.15, 4, 2)  # :62-68
    assert all(r[2] > r[i] for i in range(8) if i != 2)
    for R in (0.0, 1.0, 1.5):
        with pytest.raises(lkv.BudgetError):
            lkv.allocate_budgets(torch.zeros(8, device=DEV, dtype=torch.float64), R, 4, 2)
    with pytest.raises(lkv.ContractError):
        lkv.allocate_budgets(torch.zeros(7, device=DEV, dtype=torch.float64), 0.2, 4, 2)
    with pytest.raises(lkv.NumericError):
        lkv.budgets(torch.tensor([0.0, float("nan"), 1.0], dtype=torch.float64, device=DEV), 0.3, [100])
    with pytest.raises(lkv.OverflowGuardError):
        lkv.budgets(torch.tensor([0.0, 1e301, 1.0], dtype=torch.float64, device=DEV), 0.3, [100])
    # first offending element decides (soft_topk.cpp:61-64)
    with pytest.raises(lkv.NumericError):
        lkv.budgets(torch.tensor([0.0, float("inf"), 1e301], dtype=torch.float64, device=DEV), 0.3, [100])
    with pytest.raises(lkv.OverflowGuardError):
        lkv.budgets(torch.tensor([-1e302, float("nan"), 1.0], dtype=torch.float64, device=DEV), 0.3, [100])
    # n == 1 has no magnitude guard (soft_topk.cpp:119-131): r = clamp(R, eps, 1 - eps)
    r, b = lkv.budgets(torch.tensor([1e305], dtype=torch.float64, device=DEV), 0.3, [1000])
    assert float(r[0]) == 0.3 and int(b[0, 0]) == 300
    with pytest.raises(lkv.ContractError):
        lkv.budgets(torch.zeros(4, device=DEV, dtype=torch.float64), 0.3, [0])


def test_budget_offsets():
    logits = torch.randn(64, dtype=torch.float64, device=DEV)
    r, b, offs = lkv.budgets(logits, 0.2, [1000, 3000], lkv.BUDGET_EXACT, decode_slack=5, want_offsets=True)
    caps = (b.reshape(-1).to(torch.int64) + 5).cpu()
    want = torch.zeros(caps.numel() + 1, dtype=torch.int64)
    want[1:] = torch.cumsum(caps, 0)
    assert torch.equal(offs.cpu(), want)


# ---------------------------------------------------------------------------------------------
# K1 scorer
# ---------------------------------------------------------------------------------------------
def _oracle_scores(cache, scorers, act):
    K, V = to_np(cache.keys), to_np(cache.values)
    n_seq, L, H, T, D = cache.shape
    w1, b1, w2 = w_np(scorers.w1), w_np(scorers.b1), w_np(scorers.w2)
    out = np.zeros((n_seq, L, H, T))
    for s in range(n_seq):
        t = cache.seq_lens[s]
        for l in range(L):
            for h in range(H):
                sc = l * scorers.stride_layer + h * scorers.stride_head
                vv = V[s, l, h, :t] if scorers.input == lkv.SCORER_KV else None
                out[s, l, h, :t] = O.token_scores(K[s, l, h, :t], vv, w1[sc], b1[sc], w2[sc], act=act)
    return out


def test_scores_fp32_config1():
    cfg = synth.CONFIGS[1]
    cache = synth.make_cache(cfg)
    scorers = synth.make_scorers(cfg)
    got = lkv.token_scores(cache, scorers).cpu().numpy()
    want = _oracle_scores(cache, scorers, O.GELU_ERF)
    assert rel_gap(got, want) <= 1e-5


@pytest.mark.parametrize("inp,act,hidden", [(lkv.SCORER_K, lkv.GELU_ERF, 64), (lkv.SCORER_K, lkv.SILU, 128),
                                            (lkv.SCORER_KV, lkv.SILU, 128), (lkv.SCORER_KV, lkv.GELU_ERF, 64)])
def test_scores_bf16_tensorcore(inp, act, hidden):
    # ragged lengths (not multiples of 128), several sequences, per-(l,h) scorers
    torch.manual_seed(5)
    n_seq, L, H, T, D = 3, 2, 4, 700, 128
    K = (torch.randn(n_seq, L, H, T, D, device=DEV) * 1.5).to(torch.bfloat16)
    Vv = torch.randn(n_seq, L, H, T, D, device=DEV).to(torch.bfloat16)
    cache = lkv.DenseCache(K, Vv, [700, 129, 1])
    in_dim = inp * D
    ns = L * H
    w1 = (torch.randn(ns, in_dim, hidden, device=DEV) / math.sqrt(in_dim)).to(torch.bfloat16)
    b1 = torch.randn(ns, hidden, device=DEV) * 0.1
    w2 = torch.randn(ns, hidden, device=DEV) / math.sqrt(hidden)
    scorers = lkv.Scorers(w1, b1, w2, input=inp, activation=act, stride_layer=H, stride_head=1)
    got = lkv.token_scores(cache, scorers).cpu().numpy()
    want = _oracle_scores(cache, scorers, act)
    for s, t in enumerate(cache.seq_lens):
        assert rel_gap(got[s, :, :, :t], want[s, :, :, :t]) <= 1e-2
        assert rel_gap(got[s, :, :, :t], want[s, :, :, :t]) <= 1e-4  # fp32 accumulation: far inside the bar


def test_scores_simt_generic_shape():
    # the desk-sized reference geometry: d = 16, [k;v] -> d -> 1, SiLU (policy.cpp:101)
    torch.manual_seed(6)
    K = torch.randn(1, 2, 2, 50, 16, device=DEV)
    V = torch.randn(1, 2, 2, 50, 16, device=DEV)
    cache = lkv.DenseCache(K, V, [50])
    w1 = torch.randn(4, 32, 16, device=DEV) / math.sqrt(32)
    scorers = lkv.Scorers(w1, torch.zeros(4, 16, device=DEV), torch.randn(4, 16, device=DEV) / 4,
                          input=lkv.SCORER_KV, activation=lkv.SILU, stride_layer=2, stride_head=1)
    got = lkv.token_scores(cache, scorers).cpu().numpy()
    assert rel_gap(got, _oracle_scores(cache, scorers, O.SILU)) <= 1e-5
    # duplicate rows -> identical scores; zeros -> zero (test_policy.cpp:118-139)
    K[0, 0, 0, 4] = K[0, 0, 0, 2]
    V[0, 0, 0, 4] = V[0, 0, 0, 2]
    K[0, 0, 0, 7] = 0
    V[0, 0, 0, 7] = 0
    got = lkv.token_scores(lkv.DenseCache(K, V, [50]), scorers).cpu().numpy()
    assert got[0, 0, 0, 2] == got[0, 0, 0, 4]
    assert got[0, 0, 0, 7] == 0.0


# ---------------------------------------------------------------------------------------------
# K3 select (+ K4 gather)
# ---------------------------------------------------------------------------------------------
def _check_select(scores_np, lens, budgets_np, rc: lkv.RaggedCache, cache=None):
    offs = rc.offsets.cpu().numpy()
    pos = rc.positions.cpu().numpy()
    lens_out = rc.lens.cpu().numpy()
    n_heads = budgets_np.size
    K = to_np(cache.keys).reshape(n_heads, -1, cache.shape[-1]) if cache is not None else None
    V = to_np(cache.values).reshape(n_heads, -1, cache.shape[-1]) if cache is not None else None
    rk = to_np(rc.keys) if cache is not None else None
    rv = to_np(rc.values) if cache is not None else None
    for h in range(n_heads):
        t = lens[h]
        b = int(budgets_np[h])
        want = O.select_positions_f32(scores_np[h, :t], b)
        got = pos[offs[h]:offs[h] + b]
        assert lens_out[h] == b
        assert (got == want).all(), (h, b, t)
        if cache is not None and b:
            assert (rk[offs[h]:offs[h] + b] == K[h, want]).all()
            assert (rv[offs[h]:offs[h] + b] == V[h, want]).all()


def _select_case(scores, lens, budgets, dtype=torch.float32, D=8):
    n_heads, T = scores.shape
    K = torch.randn(1, 1, n_heads, T, D, device=DEV).to(dtype)
    V = torch.randn(1, 1, n_heads, T, D, device=DEV).to(dtype)
    assert len(set(lens)) == 1
    cache = lkv.DenseCache(K, V, [lens[0]])
    b = torch.tensor(budgets, dtype=torch.int32, device=DEV)
    rc = lkv.select(cache, scores.reshape(1, 1, n_heads, T).to(DEV), b, decode_slack=3)
    _check_select(scores.cpu().numpy(), lens, np.array(budgets), rc, cache)
    return rc


@pytest.mark.parametrize("t", [1, 2, 100, 4096, 4097, 9000, 20000])
def test_select_random(t):
    torch.manual_seed(t)
    n_heads = 6
    scores = torch.randn(n_heads, t)
    budgets = [0, 1, t // 7, t // 2, max(t - 1, 0), t]
    _select_case(scores, [t] * n_heads, budgets)


@pytest.mark.parametrize("t", [37, 4096, 10000])
def test_select_adversarial_ties(t):
    torch.manual_seed(t + 1)
    heads = [
        torch.zeros(t),                                   # all equal
        torch.randint(0, 3, (t,)).float(),                # heavy duplicates
        torch.where(torch.rand(t) < 0.5, -0.0, 0.0),      # signed zeros
        torch.randint(0, 5, (t,)).float() * 1e-30,        # denormal-scale ties
        -torch.ones(t),                                    # all negative equal
        torch.cat([torch.full((t // 2,), 3.0), torch.full((t - t // 2,), 3.0)]),
    ]
    scores = torch.stack(heads)
    for b in (0, 1, t // 3, t - 1, t):
        _select_case(scores, [t] * len(heads), [b] * len(heads))


def test_select_cluster_split_ragged():
    """Few heads (6) over ragged sequences (t = 5000 and 40000): the plan splits each head over a
    4-CTA cluster, so the short heads' clusters have CTAs without chunks; budgets 0, t, t - 1, 1 and
    interior ones, heavy ties in one head.  Indices and gathered rows vs the oracle."""
    torch.manual_seed(77)
    T, lens, D = 40000, [5000, 40000], 8
    K = torch.randn(2, 1, 3, T, D, device=DEV)
    V = torch.randn(2, 1, 3, T, D, device=DEV)
    scores = torch.randn(2, 1, 3, T)
    scores[1, 0, 2] = torch.randint(0, 4, (T,)).float()  # ties across every CTA of the cluster
    cache = lkv.DenseCache(K, V, lens)
    budgets = [[0, 5000, 1234], [1, 39999, 6000]]
    rc = lkv.select(cache, scores.to(DEV), torch.tensor(budgets, dtype=torch.int32, device=DEV).reshape(-1),
                    decode_slack=3)
    offs, pos, ln = rc.offsets.cpu().numpy(), rc.positions.cpu().numpy(), rc.lens.cpu().numpy()
    rk, Kn = to_np(rc.keys), to_np(K)
    for s in range(2):
        for h in range(3):
            i, t, b = s * 3 + h, lens[s], budgets[s][h]
            want = O.select_positions_f32(scores[s, 0, h, :t].numpy(), b)
            assert ln[i] == b
            assert (pos[offs[i]:offs[i] + b] == want).all(), (s, h)
            if b:
                assert (rk[offs[i]:offs[i] + b] == Kn[s, 0, h, want]).all()


def test_select_extreme_values():
    t = 5000
    s = torch.randn(4, t)
    s[0, ::7] = float("inf")
    s[1, ::5] = -float("inf")
    s[2] = torch.finfo(torch.float32).max
    s[3, ::3] = torch.finfo(torch.float32).tiny
    _select_case(s, [t] * 4, [10, t - 3, 77, 2500])


def test_select_errors():
    t = 300
    s = torch.randn(2, t)
    with pytest.raises(lkv.BudgetError):
        _select_case(s, [t, t], [t + 1, 3])
    with pytest.raises(lkv.BudgetError):
        _select_case(s, [t, t], [-1, 3])
    s[1, 17] = float("nan")
    with pytest.raises(lkv.NumericError):
        _select_case(s, [t, t], [5, 5])


def test_inference_select_fixtures():  # test_soft_topk.cpp:190-199 through the device path
    x = torch.tensor([0.1, 0.9, 0.5], device=DEV)
    assert lkv.inference_select(x, 2).tolist() == [0, 1, 1]
    assert lkv.inference_select(x, 0).tolist() == [0, 0, 0]
    assert lkv.inference_select(x, 3).tolist() == [1, 1, 1]
    assert lkv.inference_select(torch.tensor([0.7, 0.2, 0.7], device=DEV), 1).tolist() == [1, 0, 0]
    with pytest.raises(lkv.BudgetError):
        lkv.inference_select(x, 4)


def test_cache_from_trace_layout():  # model.cpp:289-315
    torch.manual_seed(9)
    K = torch.randn(2, 2, 2, 300, 128, device=DEV).to(torch.bfloat16)
    V = torch.randn(2, 2, 2, 300, 128, device=DEV).to(torch.bfloat16)
    cache = lkv.DenseCache(K, V, [300, 300])
    masks = (torch.rand(8, 300, device=DEV) < 0.3).to(torch.int32)
    masks[3] = 0
    masks[4] = 1
    rc = lkv.cache_from_trace(cache, masks, decode_slack=2)
    Kn, Vn = to_np(K).reshape(8, 300, 128), to_np(V).reshape(8, 300, 128)
    m = masks.cpu().numpy()
    for h in range(8):
        k, v, p = rc.head(h)
        want = np.nonzero(m[h])[0]
        assert (p.cpu().numpy() == want).all()
        assert (to_np(k) == Kn[h, want]).all() and (to_np(v) == Vn[h, want]).all()


# ---------------------------------------------------------------------------------------------
# fused eviction
# ---------------------------------------------------------------------------------------------
def _evict_and_check(cfg, cache, scorers, logits, mode):
    res = lkv.evict(cache, scorers, logits, cfg.ratio, mode, decode_slack=4, keep_scores=True)
    n_seq, L, H, T, D = cache.shape
    n = L * H
    want_r = O.allocate_budgets(logits.cpu().numpy(), cfg.ratio)
    for s, t in enumerate(cache.seq_lens):
        want_b = O.freeze_budgets(want_r, t) if mode == lkv.BUDGET_FLOOR else O.freeze_budgets_exact(want_r, cfg.ratio, t)
        assert (res.budgets[s].cpu().numpy() == want_b).all()
    scores = res.scores.reshape(n_seq * n, T).cpu().numpy()
    lens = [cache.seq_lens[h // n] for h in range(n_seq * n)]
    _check_select(scores, lens, res.budgets.reshape(-1).cpu().numpy(), res.cache, cache)
    return res


def test_evict_config1_fp32():
    cfg = synth.CONFIGS[1]
    cache = synth.make_cache(cfg)
    scorers = synth.make_scorers(cfg)
    logits = synth.make_logits(cfg)
    res = _evict_and_check(cfg, cache, scorers, logits, lkv.BUDGET_EXACT)
    assert int(res.cache.lens.sum()) == 4915
    # device scores vs the fp64 oracle
    want = _oracle_scores(cache, scorers, O.GELU_ERF)
    assert rel_gap(res.scores.cpu().numpy(), want) <= 1e-5


@pytest.mark.parametrize("cid", [2, 4, 5])
def test_evict_bf16_reduced(cid):
    cfg = synth.CONFIGS[cid]
    L, T, S = 2, 9000, (3 if cfg.n_seq > 1 else 1)
    cache = synth.make_cache(cfg, n_layers=L, max_tokens=T, n_seq=S)
    scorers = synth.make_scorers(cfg, n_layers=L)
    logits = synth.make_logits(cfg, n_layers=L)
    res = _evict_and_check(cfg, cache, scorers, logits, lkv.BUDGET_EXACT)
    want = _oracle_scores(cache, scorers, O.GELU_ERF)
    for s, t in enumerate(cache.seq_lens):
        assert rel_gap(res.scores[s, :, :, :t].cpu().numpy(), want[s, :, :, :t]) <= 1e-2
        assert int(res.budgets[s].sum()) == round(cfg.ratio * L * cfg.n_kv_heads * t)


def test_evict_floor_mode_reference_scorer():
    # reference mode end to end: [k;v] 2d -> d -> 1 SiLU, per-(l,h) scorers, floor budgets
    torch.manual_seed(12)
    L, H, T, D = 2, 4, 3000, 128
    K = torch.randn(1, L, H, T, D, device=DEV).to(torch.bfloat16)
    V = torch.randn(1, L, H, T, D, device=DEV).to(torch.bfloat16)
    cache = lkv.DenseCache(K, V, [T])
    w1 = (torch.randn(L * H, 2 * D, D, device=DEV) / math.sqrt(2 * D)).to(torch.bfloat16)
    scorers = lkv.Scorers(w1, torch.zeros(L * H, D, device=DEV), torch.randn(L * H, D, device=DEV) / math.sqrt(D),
                          input=lkv.SCORER_KV, activation=lkv.SILU, stride_layer=H, stride_head=1)
    logits = torch.randn(L * H, dtype=torch.float64, device=DEV)

    class Cfg:
        ratio = 0.15

    _evict_and_check(Cfg, cache, scorers, logits, lkv.BUDGET_FLOOR)


def test_evict_zero_and_full_budgets():
    torch.manual_seed(13)
    K = torch.randn(1, 1, 3, 500, 128, device=DEV).to(torch.bfloat16)
    cache = lkv.DenseCache(K, K.clone(), [500])
    w1 = (torch.randn(1, 128, 64, device=DEV) * 0.02).to(torch.bfloat16)
    scorers = lkv.Scorers(w1, torch.zeros(1, 64, device=DEV), torch.randn(1, 64, device=DEV) * 0.02)
    # logits that push one head to ~0 and one to ~1
    logits = torch.tensor([-40.0, 40.0, 0.0], dtype=torch.float64, device=DEV)
    res = lkv.evict(cache, scorers, logits, 0.34, lkv.BUDGET_FLOOR)
    b = res.budgets[0].cpu().tolist()
    assert b[0] == 0 and int(res.cache.lens[0]) == 0
    assert b[1] >= 499  # ratio ~ 1 - 1e-17 -> floor(r * 500) = 499 (no repair in floor mode)
    _, _, p1 = res.cache.head(1)
    p1 = p1.cpu().numpy()
    assert len(p1) == b[1] and (np.diff(p1) > 0).all()


# ---------------------------------------------------------------------------------------------
# K5 decode
# ---------------------------------------------------------------------------------------------
def _decode_oracle(rc: lkv.RaggedCache, q, n_kv, scale):
    """fp64 oracle over the device's (already appended) cache."""
    n_seq, L, Hq, D = q.shape
    G = Hq // n_kv
    qn = q.detach().to(torch.float64).cpu().numpy()
    offs = rc.offsets.cpu().numpy()
    lens = rc.lens.cpu().numpy()
    K, V = to_np(rc.keys), to_np(rc.values)
    out = np.zeros((n_seq, L, Hq, D))
    for s in range(n_seq):
        for l in range(L):
            for kvh in range(n_kv):
                h = (s * L + l) * n_kv + kvh
                rows = slice(offs[h], offs[h] + lens[h])
                out[s, l, kvh * G:(kvh + 1) * G] = O.decode_attention(qn[s, l, kvh * G:(kvh + 1) * G], K[rows],
                                                                      V[rows], scale)
    return out


@pytest.mark.parametrize("dtype,G,steps", [(torch.float32, 4, 3), (torch.bfloat16, 4, 3), (torch.bfloat16, 8, 2),
                                           (torch.bfloat16, 16, 1),
                                           # G = 16: 16 combine CTAs per head, several steps (the combine
                                           # must never see a length another CTA of the head advanced)
                                           (torch.bfloat16, 16, 5)])
def test_decode_steps(dtype, G, steps):
    torch.manual_seed(21)
    n_seq, L, H, T, D = 2, 2, 2, 1500, 128
    K = torch.randn(n_seq, L, H, T, D, device=DEV).to(dtype)
    V = torch.randn(n_seq, L, H, T, D, device=DEV).to(dtype)
    cache = lkv.DenseCache(K, V, [1500, 700])
    masks = (torch.rand(n_seq * L * H, T, device=DEV) < 0.4).to(torch.int32)
    masks[:, 700:] = masks[:, 700:] * 0  # second sequence is shorter; keep masks within t for both
    masks[1] = 0                         # a zero-budget head still attends to the new token
    masks[2, :] = 0
    masks[2, :600] = 1                   # > 2 chunks
    rc = lkv.cache_from_trace(cache, masks, decode_slack=steps + 1)
    scale = 1.0 / math.sqrt(D)
    tol = 1e-5 if dtype == torch.float32 else 1e-2
    seen0 = rc.tokens_seen.cpu().tolist()
    for step in range(steps):
        q = torch.randn(n_seq, L, H * G, D, device=DEV).to(dtype)
        nk = torch.randn(n_seq, L, H, D, device=DEV).to(dtype)
        nv = torch.randn(n_seq, L, H, D, device=DEV).to(dtype)
        lens_before = rc.lens.clone()
        out = lkv.decode_step(rc, q, nk, nv, scale)
        assert torch.equal(rc.lens, lens_before + 1)
        want = _decode_oracle(rc, q, H, scale)
        assert rel_gap(out.to(torch.float64).cpu().numpy(), want) <= tol
        # the appended row and its position are in the cache
        for h in range(n_seq * L * H):
            k, v, p = rc.head(h)
            s = h // (L * H)
            assert int(p[-1]) == seen0[s] + step
            assert torch.equal(k[-1], nk.reshape(-1, D)[h]) and torch.equal(v[-1], nv.reshape(-1, D)[h])
    assert rc.tokens_seen.cpu().tolist() == [x + steps for x in seen0]


def test_decode_capacity_exceeded():
    K = torch.randn(1, 1, 1, 64, 128, device=DEV).to(torch.bfloat16)
    cache = lkv.DenseCache(K, K.clone(), [64])
    rc = lkv.cache_from_trace(cache, torch.ones(1, 64, dtype=torch.int32, device=DEV), decode_slack=0)
    q = torch.randn(1, 1, 4, 128, device=DEV).to(torch.bfloat16)
    nk = torch.randn(1, 1, 1, 128, device=DEV).to(torch.bfloat16)
    with pytest.raises(lkv.ContractError):
        lkv.decode_step(rc, q, nk, nk, 0.1)


# ---------------------------------------------------------------------------------------------
# size-independent properties at a BASELINE size (config 2, full shape)
# ---------------------------------------------------------------------------------------------
@pytest.mark.slow
def test_config2_full_size_properties():
    cfg = synth.CONFIGS[2]
    cache = synth.make_cache(cfg)
    scorers = synth.make_scorers(cfg)
    logits = synth.make_logits(cfg)
    res = lkv.evict(cache, scorers, logits, cfg.ratio, lkv.BUDGET_EXACT, decode_slack=cfg.decode_steps,
                    keep_scores=True)
    n = cfg.n_layers * cfg.n_kv_heads
    T = cfg.max_tokens
    b = res.budgets.reshape(-1)
    assert int(b.sum()) == 1258291
    want_b = O.freeze_budgets_exact(O.allocate_budgets(logits.cpu().numpy(), cfg.ratio), cfg.ratio, T)
    assert (b.cpu().numpy() == want_b).all()
    rc = res.cache
    assert torch.equal(rc.lens.cpu(), b.cpu())
    scores = res.scores.reshape(n, T)
    offs = rc.offsets.cpu().tolist()
    Kd = cache.keys.reshape(n, T, -1)
    for h in range(n):
        bh = int(b[h])
        p = rc.positions[offs[h]:offs[h] + bh].long()
        assert bool((p[1:] > p[:-1]).all())
        mask = torch.zeros(T, dtype=torch.bool, device=DEV)
        mask[p] = True
        sel, rest = scores[h][mask], scores[h][~mask]
        if bh and rest.numel():
            lo, hi = sel.min(), rest.max()
            assert lo >= hi
            if lo == hi:  # ties: every unselected equal row lies after every selected equal row
                assert int(torch.nonzero(mask & (scores[h] == lo)).max()) < int(torch.nonzero(~mask & (scores[h] == lo)).min())
        assert torch.equal(rc.keys[offs[h]:offs[h] + bh], Kd[h][p])
        # spot-check the oracle selection on the device scores for a few heads
        if h % 37 == 0:
            assert (p.cpu().numpy() == O.select_positions_f32(scores[h].cpu().numpy(), bh)).all()


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_decode_crosses_chunk_boundaries(dtype):
    """Heads sitting just below a 256-row work-item boundary, with empty capacity-based
    items behind them: every step must plan from the same lens snapshot."""
    torch.manual_seed(23)
    L, H, T, D, G = 2, 4, 1100, 128, 4
    K = torch.randn(1, L, H, T, D, device=DEV).to(dtype)
    V = torch.randn(1, L, H, T, D, device=DEV).to(dtype)
    cache = lkv.DenseCache(K, V, [T])
    masks = torch.zeros(L * H, T, dtype=torch.int32, device=DEV)
    for h, keep in enumerate([254, 255, 256, 510, 511, 767, 1, 1023]):
        masks[h, torch.randperm(T, device=DEV)[:keep]] = 1
    rc = lkv.cache_from_trace(cache, masks, decode_slack=400)
    scale = 1.0 / math.sqrt(D)
    tol = 1e-5 if dtype == torch.float32 else 1e-2
    for step in range(4):
        q = torch.randn(1, L, H * G, D, device=DEV).to(dtype)
        nk = torch.randn(1, L, H, D, device=DEV).to(dtype)
        out = lkv.decode_step(rc, q, nk, nk * 0.5, scale)
        want = _decode_oracle(rc, q, H, scale)
        assert rel_gap(out.to(torch.float64).cpu().numpy(), want) <= tol, step


def test_decode_many_steps_stays_consistent():
    """200 steps over a C2-shaped (reduced) cache: lens, positions and outputs stay exact."""
    cfg = synth.CONFIGS[2]
    L = 2
    cache = synth.make_cache(cfg, n_layers=L, max_tokens=2000)
    scorers = synth.make_scorers(cfg, n_layers=L)
    logits = synth.make_logits(cfg, n_layers=L)
    res = lkv.evict(cache, scorers, logits, cfg.ratio, lkv.BUDGET_EXACT, decode_slack=200)
    rc = res.cache
    lens0 = rc.lens.clone()
    for s in range(200):
        q, k, v = synth.make_decode_inputs(cfg, s, n_layers=L)
        out = lkv.decode_step(rc, q, k, v, check=(s % 50 == 49))
    assert torch.equal(rc.lens, lens0 + 200)
    assert int(rc.tokens_seen[0]) == 2000 + 200
    want = _decode_oracle(rc, q, cfg.n_kv_heads, 1 / math.sqrt(cfg.head_dim))
    assert rel_gap(out.to(torch.float64).cpu().numpy(), want) <= 1e-2
    for h in range(L * cfg.n_kv_heads):
        _, _, p = rc.head(h)
        p = p.cpu().numpy()
        assert (np.diff(p) > 0).all() and p[-1] == 2000 + 199


@pytest.mark.parametrize("cid,inp,chunk", [(2, lkv.SCORER_K, 2), (4, lkv.SCORER_K, 2), (2, lkv.SCORER_KV, 2),
                                            (1, lkv.SCORER_K, 1), (4, lkv.SCORER_K, 3), (4, lkv.SCORER_K, 5)])
def test_evict_from_host_memory_matches_device_path(cid, inp, chunk):
    """lkv_evict_host (per-chunk pipeline: K streamed in, scored, selected, kept V gathered over
    PCIe from pinned host memory, chunk copied back while later chunks upload) produces exactly
    the device-resident eviction, for chunkings that split, cover and exceed the layer count."""
    cfg = synth.CONFIGS[cid]
    L, T, S = 3, 5000, (3 if cfg.n_seq > 1 else 1)
    cache = synth.make_cache(cfg, n_layers=L, max_tokens=T, n_seq=S)
    if inp == lkv.SCORER_KV:
        w1 = (torch.randn(L * 8, 256, 128, device=DEV) / 16).to(torch.bfloat16)
        scorers = lkv.Scorers(w1, torch.zeros(L * 8, 128, device=DEV), torch.randn(L * 8, 128, device=DEV) / 11,
                              input=lkv.SCORER_KV, activation=lkv.SILU, stride_layer=8, stride_head=1)
    else:
        scorers = synth.make_scorers(cfg, n_layers=L)
    logits = synth.make_logits(cfg, n_layers=L)
    ref = lkv.evict(cache, scorers, logits, cfg.ratio, lkv.BUDGET_EXACT, decode_slack=2, keep_scores=False)
    hk = cache.keys.cpu().pin_memory()
    hv = cache.values.cpu().pin_memory()
    dense = lkv.DenseCache(torch.zeros_like(cache.keys), torch.zeros_like(cache.values), cache.seq_lens)
    ev = lkv.Evictor(dense, scorers, logits, cfg.ratio, lkv.BUDGET_EXACT, decode_slack=2)
    out = ev.host_result_buffer()
    ev.launch_host(hk, hv, out, layers_per_chunk=chunk)
    ev.ws.status()
    torch.cuda.synchronize()
    assert torch.equal(ev.ragged.lens, ref.cache.lens)
    assert torch.equal(out.lens, ref.cache.lens.cpu())
    assert torch.equal(out.offsets, ref.cache.offsets.cpu())
    for h in range(cache.n_heads):
        o, n = int(out.offsets[h]), int(out.lens[h])
        ko, vo, po = ref.cache.head(h)
        assert torch.equal(out.positions[o:o + n], po.cpu())
        assert torch.equal(out.keys[o:o + n], ko.cpu()) and torch.equal(out.values[o:o + n], vo.cpu())


def test_evict_from_host_memory_without_copy_back():
    """host_out = NULL: the compacted cache stays on the device, identical to lkv_evict's."""
    cfg = synth.CONFIGS[2]
    cache = synth.make_cache(cfg, n_layers=5, max_tokens=3000)
    scorers = synth.make_scorers(cfg, n_layers=5)
    logits = synth.make_logits(cfg, n_layers=5)
    ref = lkv.evict(cache, scorers, logits, cfg.ratio, lkv.BUDGET_EXACT, decode_slack=1)
    dense = lkv.DenseCache(torch.zeros_like(cache.keys), torch.zeros_like(cache.values), cache.seq_lens)
    ev = lkv.Evictor(dense, scorers, logits, cfg.ratio, lkv.BUDGET_EXACT, decode_slack=1)
    ev.launch_host(cache.keys.cpu().pin_memory(), cache.values.cpu().pin_memory(), None, layers_per_chunk=2)
    ev.ws.status()
    torch.cuda.synchronize()
    assert torch.equal(ev.ragged.offsets, ref.cache.offsets) and torch.equal(ev.ragged.lens, ref.cache.lens)
    for h in range(cache.n_heads):
        k, v, p = ev.ragged.head(h)
        ko, vo, po = ref.cache.head(h)
        assert torch.equal(p, po) and torch.equal(k, ko) and torch.equal(v, vo)


def test_evict_is_deterministic():
    """Two evictions of the same inputs are byte-identical (the reference's rerun determinism,
    test_distill.cpp:251-259): scores, budgets, positions and rows."""
    cfg = synth.CONFIGS[4]
    cache = synth.make_cache(cfg, n_layers=2, max_tokens=6000, n_seq=3)
    scorers = synth.make_scorers(cfg, n_layers=2)
    logits = synth.make_logits(cfg, n_layers=2)
    a = lkv.evict(cache, scorers, logits, cfg.ratio, lkv.BUDGET_EXACT, decode_slack=1)
    b = lkv.evict(cache, scorers, logits, cfg.ratio, lkv.BUDGET_EXACT, decode_slack=1)
    assert torch.equal(a.scores, b.scores) and torch.equal(a.budgets, b.budgets)
    assert torch.equal(a.cache.offsets, b.cache.offsets) and torch.equal(a.cache.lens, b.cache.lens)
    cap = int(a.cache.offsets[-1])
    for x, y in ((a.cache.positions, b.cache.positions), (a.cache.keys, b.cache.keys), (a.cache.values, b.cache.values)):
        for h in range(cache.n_heads):
            o, n = int(a.cache.offsets[h]), int(a.cache.lens[h])
            assert torch.equal(x[o:o + n], y[o:o + n])
    assert cap == int(b.cache.offsets[-1])


@pytest.mark.slow
@pytest.mark.parametrize("ratio", [0.05, 0.10, 0.25])
def test_config3_full_size_properties(ratio):
    """C3 at full size (t = 131072, 256 heads): exact totals, top-b property with the
    lowest-index tie rule, rows equal the dense rows at the kept positions."""
    cfg = synth.CONFIGS[3]
    cache = synth.make_cache(cfg)
    scorers = synth.make_scorers(cfg)
    logits = synth.make_logits(cfg)
    res = lkv.evict(cache, scorers, logits, ratio, lkv.BUDGET_EXACT, keep_scores=True)
    n, T = cfg.n_layers * cfg.n_kv_heads, cfg.max_tokens
    b = res.budgets.reshape(-1)
    assert int(b.sum()) == {0.05: 1677722, 0.10: 3355443, 0.25: 8388608}[ratio]
    want_b = O.freeze_budgets_exact(O.allocate_budgets(logits.cpu().numpy(), ratio), ratio, T)
    assert (b.cpu().numpy() == want_b).all()
    scores = res.scores.reshape(n, T)
    offs = res.cache.offsets.cpu().tolist()
    Kd = cache.keys.reshape(n, T, -1)
    Vd = cache.values.reshape(n, T, -1)
    for h in range(n):
        bh = int(b[h])
        p = res.cache.positions[offs[h]:offs[h] + bh].long()
        assert bool((p[1:] > p[:-1]).all())
        mask = torch.zeros(T, dtype=torch.bool, device=DEV)
        mask[p] = True
        sel, rest = scores[h][mask], scores[h][~mask]
        if bh and rest.numel():
            assert sel.min() >= rest.max()
        assert torch.equal(res.cache.keys[offs[h]:offs[h] + bh], Kd[h][p])
        assert torch.equal(res.cache.values[offs[h]:offs[h] + bh], Vd[h][p])
        if h % 61 == 0:
            assert (p.cpu().numpy() == O.select_positions_f32(scores[h].cpu().numpy(), bh)).all()


@pytest.mark.slow
def test_config3_headline_full_parity():
    """The bench's headline workload, C3 at full size (t = 131072, 32 x 8 heads, R = 0.15, exact
    budgets, one lkv_evict): budgets bit-exact (total 5,033,165); EVERY head's kept positions
    bit-exact against the oracle's stable-sort top-k on the device scores; every kept K/V row equal
    to the dense row; K1 scores within 1e-2 of the fp64 oracle on 8 full heads spread over the
    layers; then decode over that cache with the bench's 1024-row work items, checked against the
    fp64 oracle on sampled heads (the largest heads included)."""
    cfg = synth.CONFIGS[3]
    cache = synth.make_cache(cfg)
    scorers = synth.make_scorers(cfg)
    logits = synth.make_logits(cfg)
    res = lkv.evict(cache, scorers, logits, 0.15, lkv.BUDGET_EXACT, decode_slack=4, keep_scores=True)
    n, T, D = cfg.n_layers * cfg.n_kv_heads, cfg.max_tokens, cfg.head_dim
    b = res.budgets.reshape(-1).cpu().numpy()
    assert int(b.sum()) == 5033165
    want_b = O.freeze_budgets_exact(O.allocate_budgets(logits.cpu().numpy(), 0.15), 0.15, T)
    assert (b == want_b).all()
    rc = res.cache
    offs = rc.offsets.cpu().numpy()
    assert (rc.lens.cpu().numpy() == b).all()
    scores = res.scores.reshape(n, T).cpu().numpy()
    pos_all = rc.positions.cpu().numpy()
    Kd = cache.keys.reshape(n, T, D)
    Vd = cache.values.reshape(n, T, D)
    for h in range(n):
        bh = int(b[h])
        p = pos_all[offs[h]:offs[h] + bh]
        assert (p == O.select_positions_f32(scores[h], bh)).all(), h
        pt = torch.from_numpy(p.astype(np.int64)).to(DEV)
        assert torch.equal(rc.keys[offs[h]:offs[h] + bh], Kd[h][pt]), h
        assert torch.equal(rc.values[offs[h]:offs[h] + bh], Vd[h][pt]), h
    # K1 scores at full length on 8 heads (layers 0, 4, ..., 28; head l % 8)
    w1 = w_np(scorers.w1)
    for l in range(0, cfg.n_layers, 4):
        h = l * cfg.n_kv_heads + (l % cfg.n_kv_heads)
        ref = O.token_scores(to_np(Kd[h]), None, w1[l], w_np(scorers.b1[l]), w_np(scorers.w2[l]), act=O.GELU_ERF)
        assert rel_gap(scores[h], ref) <= 1e-2, h
    # decode with the measured work-item size (all layers per launch, ch = 1024)
    G = cfg.n_q_heads // cfg.n_kv_heads
    rc.tokens_seen.fill_(T)
    lkv.decode_plan(rc, G, rows_per_item=1024)
    assert lkv.decode_plan_info(rc)[1] == 1024
    del res, scores
    for st in range(2):
        q, k, v = synth.make_decode_inputs(cfg, st)
        out = lkv.decode_step(rc, q, k, v)
    heads = sorted(set([int(np.argmax(b)), int(np.argmin(b))] + list(range(0, n, 23))))
    _check_decode_heads(rc, q, out, cfg.n_kv_heads, heads, 1e-2)


def _check_decode_heads(rc, q, out, n_kv, heads, tol):
    """fp64 oracle over the device's cache for the listed flat heads (n_seq == 1)."""
    _, L, Hq, D = q.shape
    G = Hq // n_kv
    scale = 1.0 / math.sqrt(D)
    qn = q.detach().to(torch.float64).cpu().numpy()
    on = out.detach().to(torch.float64).cpu().numpy()
    offs = rc.offsets.cpu().numpy()
    lens = rc.lens.cpu().numpy()
    for h in heads:
        l, kvh = divmod(h, n_kv)
        o, ln = int(offs[h]), int(lens[h])
        want = O.decode_attention(qn[0, l, kvh * G:(kvh + 1) * G], to_np(rc.keys[o:o + ln]), to_np(rc.values[o:o + ln]),
                                  scale)
        assert rel_gap(on[0, l, kvh * G:(kvh + 1) * G], want) <= tol, h


@pytest.mark.slow
@pytest.mark.parametrize("rows_per_item", [0, 1024, 192])
def test_config2_full_size_decode_work_items(rows_per_item):
    """Decode over the full evicted C2 cache with the work-item size the bench measures (the
    automatic all-layer plan picks 1024 rows here) and two forced sizes, against the fp64 oracle on
    every head."""
    cfg = synth.CONFIGS[2]
    cache = synth.make_cache(cfg)
    res = lkv.evict(cache, synth.make_scorers(cfg), synth.make_logits(cfg), cfg.ratio, lkv.BUDGET_EXACT,
                    decode_slack=8)
    del cache
    rc = res.cache
    rc.tokens_seen.fill_(cfg.max_tokens)
    G = cfg.n_q_heads // cfg.n_kv_heads
    lkv.decode_plan(rc, G, rows_per_item=rows_per_item)
    n_items, ch = lkv.decode_plan_info(rc)
    assert ch == (rows_per_item or 1024)
    assert n_items >= rc.n_heads
    for st in range(3):
        q, k, v = synth.make_decode_inputs(cfg, st)
        out = lkv.decode_step(rc, q, k, v)
    want = _decode_oracle(rc, q, cfg.n_kv_heads, 1.0 / math.sqrt(cfg.head_dim))
    assert rel_gap(out.to(torch.float64).cpu().numpy(), want) <= 1e-2


def test_compact_rejects_out_of_range_positions():
    """lkv_compact: a position outside [0, t) is a contract_error, latched in the workspace; the
    head's rows are not written (never replaced by another row)."""
    torch.manual_seed(3)
    K = torch.randn(1, 1, 2, 64, 128, device=DEV).to(torch.bfloat16)
    cache = lkv.DenseCache(K, K.clone(), [64])
    rc = lkv.RaggedCache(1, 1, 2, 128, torch.bfloat16, 8, 0)
    rc.offsets.copy_(torch.tensor([0, 4, 8], dtype=torch.int64))
    rc.lens.fill_(4)
    rc.positions.copy_(torch.tensor([0, 5, 9, 63, 1, 2, 64, 3], dtype=torch.int32))
    rc.keys.fill_(7.0)
    with pytest.raises(lkv.ContractError):
        lkv.compact(cache, rc)
    assert torch.equal(rc.keys[:4], K[0, 0, 0][[0, 5, 9, 63]])
    assert bool((rc.keys[4:] == 7.0).all())  # head 1 (position 64 >= t) untouched
    rc.positions[6] = 4
    lkv.compact(cache, rc)
    assert torch.equal(rc.keys[4:], K[0, 0, 1][[1, 2, 4, 3]])


def test_cache_from_trace_capacity_and_ragged_lengths():
    """Device mask scan over ragged sequences (t_s < max_tokens, heads longer than one 4096-row
    chunk): counts, offsets (with decode slack), positions and rows exact."""
    torch.manual_seed(4)
    T = 9000
    K = torch.randn(2, 1, 2, T, 128, device=DEV).to(torch.bfloat16)
    V = torch.randn(2, 1, 2, T, 128, device=DEV).to(torch.bfloat16)
    cache = lkv.DenseCache(K, V, [T, 5000])
    masks = (torch.rand(4, T, device=DEV) < 0.2).to(torch.int32)
    masks[2:, 5000:] = 1  # past t_s: never kept
    rc = lkv.cache_from_trace(cache, masks, decode_slack=3)
    m = masks.cpu().numpy()
    offs = rc.offsets.cpu().numpy()
    Kn, Vn = to_np(K).reshape(4, T, 128), to_np(V).reshape(4, T, 128)
    for h in range(4):
        t = T if h < 2 else 5000
        want = np.nonzero(m[h, :t])[0]
        k, v, p = rc.head(h)
        assert (p.cpu().numpy() == want).all()
        assert offs[h + 1] - offs[h] == len(want) + 3
        assert (to_np(k) == Kn[h, want]).all() and (to_np(v) == Vn[h, want]).all()


# ---------------------------------------------------------------------------------------------
# layer-by-layer prefill
# ---------------------------------------------------------------------------------------------
def test_rope_pack_matches_fp64_rope():  # tensor.cpp:586-623 convention, absolute positions
    from paper_2605_06676_b200 import prefill

    torch.manual_seed(41)
    S, T, H, D = 2, 600, 3, 128
    for dtype, tol in ((torch.float32, 1e-5), (torch.bfloat16, 1e-2)):
        k_lin = torch.randn(S, T, H * D, device=DEV).to(dtype)
        v_lin = torch.randn(S, T, H * D, device=DEV).to(dtype)
        tab = prefill.rope_table(T, D)
        k, v = prefill.rope_pack(k_lin, v_lin, tab, [T, 450], H)
        kl = k_lin.double().cpu().numpy().reshape(S, T, H, D)
        pos = np.arange(T)[:, None]
        freq = 10000.0 ** (-2.0 * np.arange(D // 2) / D)
        th = pos * freq[None, :]
        a, b = kl[..., 0::2], kl[..., 1::2]
        want = np.empty_like(kl)
        want[..., 0::2] = a * np.cos(th)[None, :, None, :] - b * np.sin(th)[None, :, None, :]
        want[..., 1::2] = a * np.sin(th)[None, :, None, :] + b * np.cos(th)[None, :, None, :]
        got = k.double().cpu().numpy()[:, 0].transpose(0, 2, 1, 3)
        assert rel_gap(got[0], want[0]) <= tol and rel_gap(got[1, :450], want[1, :450]) <= tol
        assert torch.equal(v[:, 0].transpose(1, 2).reshape(S, T, H * D)[1, :450], v_lin[1, :450])


@pytest.mark.parametrize("S,T,H,dm", [(2, 300, 2, 256), (1, 1024, 8, 512), (3, 129, 4, 64),
                                     (1, 20000, 8, 256), (2, 9000, 4, 1024),  # these two: many tiles per pair
                                     (1, 100, 1, 64), (1, 256, 1, 128)])  # one 256-row pair tile: partial / exact
def test_kv_project_matches_fp64_projection_and_rope(S, T, H, dm):
    """lkv_kv_project (tcgen05 GEMM on CTA pairs, RoPE + head-major pack in the epilogue) vs the fp64 oracle of
    evictsim.cpp:133-145: k = rope(h Wk) at absolute positions, v = h Wv, on the same bf16 inputs;
    bf16 bar 1e-2 (observed ~3e-3: fp32 accumulation, one bf16 rounding of the output).  Token
    counts off the 128-row tile, several heads per 256-column tile."""
    from paper_2605_06676_b200 import prefill

    torch.manual_seed(S * 1000 + T)
    D = 128
    h = (torch.randn(S, T, dm, device=DEV) * 0.5).to(torch.bfloat16)
    wk = (torch.randn(dm, H * D, device=DEV) / math.sqrt(dm)).to(torch.bfloat16)
    wv = (torch.randn(dm, H * D, device=DEV) / math.sqrt(dm)).to(torch.bfloat16)
    tab = prefill.rope_table(T, D)
    k, v = prefill.kv_project(h, prefill.kv_weights(wk, wv), tab, [T] * S, H)
    hd = h.double().cpu().numpy()
    kl = (hd @ wk.double().cpu().numpy()).reshape(S, T, H, D)
    vl = (hd @ wv.double().cpu().numpy()).reshape(S, T, H, D)
    pos = np.arange(T)[:, None]
    th = pos * (10000.0 ** (-2.0 * np.arange(D // 2) / D))[None, :]
    a, b = kl[..., 0::2], kl[..., 1::2]
    want_k = np.empty_like(kl)
    want_k[..., 0::2] = a * np.cos(th)[None, :, None, :] - b * np.sin(th)[None, :, None, :]
    want_k[..., 1::2] = a * np.sin(th)[None, :, None, :] + b * np.cos(th)[None, :, None, :]
    got_k = k.double().cpu().numpy()[:, 0].transpose(0, 2, 1, 3)
    got_v = v.double().cpu().numpy()[:, 0].transpose(0, 2, 1, 3)
    assert rel_gap(got_k, want_k) <= 1e-2
    assert rel_gap(got_v, vl) <= 1e-2


def test_layerwise_prefill_from_hidden_states_equals_one_shot():
    """Layer-by-layer prefill fed by lkv_kv_project (ingest_layer_hidden) == one lkv_evict over the
    dense cache that the same kernel produces layer by layer: budgets, offsets, positions and rows
    bit-exact."""
    from paper_2605_06676_b200 import prefill

    cfg = synth.CONFIGS[2]
    S, L, H, D, T, dm = 1, 3, 8, 128, 2000, 512
    torch.manual_seed(77)
    hs = [(torch.randn(S, T, dm, device=DEV) * 0.5).to(torch.bfloat16) for _ in range(L)]
    ws = [prefill.kv_weights((torch.randn(dm, H * D, device=DEV) / math.sqrt(dm)).to(torch.bfloat16),
                             (torch.randn(dm, H * D, device=DEV) / math.sqrt(dm)).to(torch.bfloat16)) for _ in range(L)]
    scorers = synth.make_scorers(cfg, n_layers=L)
    logits = synth.make_logits(cfg, n_layers=L)
    pf = prefill.LayerwisePrefill(S, L, H, D, T, [T], scorers, logits, cfg.ratio, lkv.BUDGET_EXACT, decode_slack=2)
    for l in range(L):
        pf.ingest_layer_hidden(l, hs[l], ws[l])
    rc = pf.finish()
    tab = prefill.rope_table(T, D)
    K = torch.empty(S, L, H, T, D, dtype=torch.bfloat16, device=DEV)
    V = torch.empty_like(K)
    for l in range(L):
        k, v = prefill.kv_project(hs[l], ws[l], tab, [T], H)
        K[:, l], V[:, l] = k[:, 0], v[:, 0]
    ref = lkv.evict(lkv.DenseCache(K, V, [T]), scorers, logits, cfg.ratio, lkv.BUDGET_EXACT, decode_slack=2)
    assert torch.equal(rc.offsets, ref.cache.offsets) and torch.equal(rc.lens, ref.cache.lens)
    for i in range(L * H):
        assert all(torch.equal(a, b) for a, b in zip(rc.head(i), ref.cache.head(i))), i


def test_rope_pack_noncontiguous_views():
    """rope_pack on strided views (k and v slices of one [T, 2HD] projection): each gets its own
    contiguous copy for the duration of the call (two temporaries freed inside one argument list
    used to share a caching-allocator block, so K came out as rope(V))."""
    from paper_2605_06676_b200 import prefill

    torch.manual_seed(43)
    S, T, H, D = 1, 700, 2, 128
    kv = torch.randn(S, T, 2 * H * D, device=DEV).to(torch.bfloat16)
    tab = prefill.rope_table(T, D)
    k1, v1 = prefill.rope_pack(kv[..., :H * D], kv[..., H * D:], tab, [T], H)
    k2, v2 = prefill.rope_pack(kv[..., :H * D].contiguous(), kv[..., H * D:].contiguous(), tab, [T], H)
    assert torch.equal(k1, k2) and torch.equal(v1, v2)


def test_layerwise_prefill_equals_one_shot_eviction():
    """Per-layer rope + score + select into one ragged cache == one lkv_evict over the whole
    dense cache; peak KV = one dense layer + the compressed earlier layers (evictsim.cpp:157-159)."""
    from paper_2605_06676_b200 import prefill

    torch.manual_seed(43)
    S, L, H, D, T, dm = 2, 3, 4, 128, 3000, 256
    cfg = synth.CONFIGS[2]
    lens = [T, 2100]
    x = torch.randn(S, T, dm, device=DEV).to(torch.bfloat16)
    wk = [(torch.randn(dm, H * D, device=DEV) / dm ** 0.5).to(torch.bfloat16) for _ in range(L)]
    wv = [(torch.randn(dm, H * D, device=DEV) / dm ** 0.5).to(torch.bfloat16) for _ in range(L)]
    w1 = (torch.randn(L, D, 64, device=DEV) * 0.05).to(torch.bfloat16)
    scorers = lkv.Scorers(w1, torch.zeros(L, 64, device=DEV), torch.randn(L, 64, device=DEV) * 0.05)
    logits = torch.randn(L * H, dtype=torch.float64, device=DEV)
    pf = prefill.LayerwisePrefill(S, L, H, D, T, lens, scorers, logits, 0.2, lkv.BUDGET_EXACT, decode_slack=3)
    K = torch.empty(S, L, H, T, D, dtype=torch.bfloat16, device=DEV)
    V = torch.empty_like(K)
    for l in range(L):
        k_lin, v_lin = x @ wk[l], x @ wv[l]          # cuBLAS projections
        pf.ingest_layer(l, k_lin, v_lin)
        K[:, l], V[:, l] = (t[:, 0] for t in prefill.rope_pack(k_lin, v_lin, pf.table, lens, H))
    rc = pf.finish()
    ref = lkv.evict(lkv.DenseCache(K, V, lens), scorers, logits, 0.2, lkv.BUDGET_EXACT, decode_slack=3)
    assert torch.equal(rc.offsets, ref.cache.offsets) and torch.equal(rc.lens, ref.cache.lens)
    for h in range(S * L * H):
        a, b = rc.head(h), ref.cache.head(h)
        assert all(torch.equal(u, w) for u, w in zip(a, b)), h
    dense_layer = 2 * S * H * T * D * 2
    compressed_before_last = int(ref.budgets.reshape(S, L, H)[:, :L - 1].sum()) * 2 * D * 2
    assert pf.peak_kv_bytes == dense_layer + compressed_before_last


@pytest.mark.gpu
def test_evict_graph_replay_matches_eager():
    """lkv_evict captured in a CUDA graph (its K2 -> K1 -> plan -> emit programmatic-dependent
    chain is captured as such) and replayed gives the eager result, also after the logits change
    between replays (budgets re-solved inside the graph)."""
    cfg = synth.CONFIGS[2]
    cache = synth.make_cache(cfg, n_layers=2, max_tokens=8192)
    scorers = synth.make_scorers(cfg, n_layers=2)
    ev = lkv.Evictor(cache, scorers, synth.make_logits(cfg, n_layers=2), cfg.ratio, lkv.BUDGET_EXACT,
                     decode_slack=1)

    def snapshot():
        r = ev.ragged
        return (ev.budgets.clone(), r.offsets.clone(), r.lens.clone(), r.positions.clone(), r.keys.clone(),
                r.values.clone())

    ev.launch()
    torch.cuda.synchronize()
    ev.ws.status()
    eager = snapshot()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        ev.launch(s)  # warm-up on the capture stream
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            ev.launch(s)
    def same(x, y):  # budgets / offsets / lens in full, rows and positions over each head's kept range
        for a, b in zip(x[:3], y[:3]):
            assert torch.equal(a, b)
        for h in range(cache.n_heads):
            o, n = int(x[1][h]), int(x[2][h])
            for a, b in zip(x[3:], y[3:]):
                assert torch.equal(a[o:o + n], b[o:o + n])

    for _ in range(2):
        ev.ragged.positions.zero_()
        ev.ragged.keys.zero_()
        g.replay()
        torch.cuda.synchronize()
        ev.ws.status()
        same(eager, snapshot())
    ev.logits.copy_(ev.logits.flip(0))  # new LKV-H logits: the replay re-solves the budgets
    g.replay()
    torch.cuda.synchronize()
    ev.ws.status()
    replayed = snapshot()
    ev.launch()
    torch.cuda.synchronize()
    ev.ws.status()
    eager2 = snapshot()
    assert not torch.equal(eager2[0], eager[0])
    same(eager2, replayed)
