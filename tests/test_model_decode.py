"""Full decode step of the toy GQA model on the B200 vs the fp64 oracle
(oracle/model.py, itself pinned against the reference's model.cpp in tests/test_oracle.py) and,
where oracle/_ref is present, vs the reference's own decode_step.

Bars: fp32 models 1e-5, bf16 models 1e-2 (rel_gap = max|d| / max|ref|, gradcheck.cpp:74-81);
positions, lens and tokens_seen exact.  The oracle is fed the device's own rounded weights and
cache rows, so the gap measures the step's arithmetic only."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle as O
import paper_2605_06676_b200 as lkv
from oracle import model as OM
from paper_2605_06676_b200 import model as M

pytestmark = pytest.mark.gpu
DEV = "cuda"


def rel_gap(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / (np.abs(b).max() + 1e-12))


def _round(P, dtype):
    """The params as the device holds them (dtype-rounded), back in fp64."""
    return {k: torch.as_tensor(v).to(dtype).double().numpy() for k, v in P.items()}


def _caches(cfg, P, n_seq, t, seed, keep=0.5):
    """Per sequence: the oracle's prefill K/V over t random tokens, random retention masks."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n_seq):
        toks = rng.integers(0, cfg.vocab_size, t)
        _, K, V = OM.forward_full(cfg, P, toks)
        heads = []
        for i in range(cfg.total_kv_heads):
            idx = np.nonzero(rng.random(t) < keep)[0]
            heads.append(OM.HeadCache(K[i][idx], V[i][idx], idx.astype(np.int32)))
        out.append(heads)
    return out


def _ragged(cfg, seqs, dtype, slack, t):
    """RaggedCache holding every sequence's heads (flat head (s * L + l) * H + h); returns it and
    the oracle heads rewritten with the device-rounded rows."""
    S, n = len(seqs), cfg.total_kv_heads
    lens = [len(h.positions) for hs in seqs for h in hs]
    caps = [x + slack for x in lens]
    offs = np.zeros(S * n + 1, np.int64)
    offs[1:] = np.cumsum(caps)
    rc = lkv.RaggedCache(S, cfg.n_layers, cfg.n_kv_heads, cfg.head_dim, dtype, int(offs[-1]), slack)
    K = torch.zeros(int(offs[-1]), cfg.head_dim, dtype=torch.float64)
    V = torch.zeros_like(K)
    pos = torch.full((int(offs[-1]),), -1, dtype=torch.int32)
    for i, h in enumerate(h for hs in seqs for h in hs):
        o = int(offs[i])
        K[o:o + lens[i]] = torch.from_numpy(h.keys.reshape(-1, cfg.head_dim))
        V[o:o + lens[i]] = torch.from_numpy(h.values.reshape(-1, cfg.head_dim))
        pos[o:o + lens[i]] = torch.from_numpy(h.positions)
    rc.offsets.copy_(torch.from_numpy(offs))
    rc.lens.copy_(torch.tensor(lens, dtype=torch.int32))
    rc.keys.copy_(K.to(dtype))
    rc.values.copy_(V.to(dtype))
    rc.positions.copy_(pos)
    rc.tokens_seen.fill_(t)
    Kr, Vr = rc.keys.double().cpu().numpy(), rc.values.double().cpu().numpy()
    rounded = []
    for s, hs in enumerate(seqs):
        rr = []
        for j, h in enumerate(hs):
            i = s * n + j
            o = int(offs[i])
            rr.append(OM.HeadCache(Kr[o:o + lens[i]].copy(), Vr[o:o + lens[i]].copy(), h.positions.copy()))
        rounded.append(rr)
    return rc, rounded


def _run(cfg, P, dtype, n_seq, t, steps, seed, tol, slack=None, rows_per_item=0):
    torch.manual_seed(seed)
    Pd = _round(P, dtype)
    seqs = _caches(cfg, Pd, n_seq, t, seed)
    slack = steps + 2 if slack is None else slack
    rc, ref_heads = _ragged(cfg, seqs, dtype, slack, t)
    lens0 = rc.lens.clone()
    dm = M.DecodeModel(M.ModelConfig(**{k: getattr(cfg, k) for k in ("n_layers", "n_query_heads", "n_kv_heads",
                                                                      "head_dim", "vocab_size", "max_seq_len",
                                                                      "mlp_hidden")}), P, dtype=dtype)
    dm.bind(rc, rows_per_item=rows_per_item)
    if rows_per_item:
        assert lkv.decode_plan_info(rc, dm.ws)[1] == rows_per_item
    rng = np.random.default_rng(seed + 1)
    for step in range(steps):
        toks = rng.integers(0, cfg.vocab_size, n_seq)
        lg = dm.step(torch.tensor(toks, dtype=torch.int32, device=DEV)).cpu().numpy()
        for s in range(n_seq):
            want, seen = OM.decode_step(cfg, Pd, ref_heads[s], t + step, int(toks[s]))
            assert rel_gap(lg[s], want) <= tol, (step, s, rel_gap(lg[s], want))
        # the appended rows: keys/values vs the oracle's, positions exact
        for s in range(n_seq):
            for j in range(cfg.total_kv_heads):
                i = s * cfg.total_kv_heads + j
                o, n = int(rc.offsets[i]), int(rc.lens[i])
                assert n == int(lens0[i]) + step + 1
                assert int(rc.positions[o + n - 1]) == t + step
                kd = rc.keys[o + n - 1].double().cpu().numpy()
                vd = rc.values[o + n - 1].double().cpu().numpy()
                h = ref_heads[s][j]
                assert np.abs(kd - h.keys[-1]).max() <= tol * max(np.abs(h.keys[-1]).max(), 1e-3) * 4
                assert np.abs(vd - h.values[-1]).max() <= tol * max(np.abs(h.values[-1]).max(), 1e-3) * 4
                # the oracle continues from the device's rounded row (as the device does)
                h.keys[-1], h.values[-1] = kd, vd
        assert rc.tokens_seen.cpu().tolist() == [t + step + 1] * n_seq
    return dm, rc


def test_model_decode_f32_reference_toy_config():
    """The reference's default toy geometry (model.hpp:18-26: L=4, Hq=8, H=2, d=16, vocab=256),
    fp32, 2 sequences, 3 steps; weights from the reference-distribution init."""
    cfg = OM.ModelConfig()
    P = OM.random_params(cfg, 5, norm_jitter=0.1)
    _run(cfg, P, torch.float32, n_seq=2, t=40, steps=3, seed=7, tol=1e-5)


def test_model_decode_f32_ragged_dims():
    """Shapes off every tile boundary: d_model 96, H*d 48, mlp 200, vocab 1000 (column groups
    of 64 and k-units of 128 both cut)."""
    cfg = OM.ModelConfig(n_layers=2, n_query_heads=6, n_kv_heads=3, head_dim=16, vocab_size=1000, max_seq_len=100,
                         mlp_hidden=200)
    P = OM.random_params(cfg, 6, gain=0.1, norm_jitter=0.1)
    _run(cfg, P, torch.float32, n_seq=3, t=30, steps=2, seed=8, tol=1e-5)


@pytest.mark.parametrize("n_seq", [1, 3, 9, 16])
def test_model_decode_bf16(n_seq):
    """bf16, d=128 (the tensor-core attention envelope), G=4; B=9/16 use two batch tiles."""
    cfg = OM.ModelConfig(n_layers=2, n_query_heads=8, n_kv_heads=2, head_dim=128, vocab_size=1000, max_seq_len=512)
    P = OM.random_params(cfg, 9, norm_jitter=0.1)
    _run(cfg, P, torch.bfloat16, n_seq=n_seq, t=200 if n_seq < 9 else 64, steps=2, seed=10 + n_seq, tol=1e-2)


@pytest.mark.parametrize("rows_per_item", [0, 512, 1024, 192])
def test_model_decode_bf16_gqa8_long_cache(rows_per_item):
    """G=8, ~1500-row heads: the one-wave plan (0 picks the smallest 64-multiple that fits one
    wave, 128 rows for these four heads) and forced 512 / 1024 / 192-row work items, i.e. heads
    spanning 1-3 large chunks and the multi-slice combine."""
    cfg = OM.ModelConfig(n_layers=1, n_query_heads=16, n_kv_heads=2, head_dim=128, vocab_size=300,
                         max_seq_len=4096, mlp_hidden=512)
    P = OM.random_params(cfg, 12, norm_jitter=0.1)
    _run(cfg, P, torch.bfloat16, n_seq=2, t=3000, steps=2, seed=13, tol=1e-2, slack=5, rows_per_item=rows_per_item)


@pytest.mark.parametrize("n_seq", [1, 5, 16])
def test_model_decode_bf16_wide_gemv_paths(n_seq):
    """d_model 2048, G = 4, mlp 14336: the launch rules the Llama-3-8B step takes -- QKV (48 column
    groups) and Wo / down (32) as split-K clusters with the DSMEM tail (one output per thread at
    n_seq 1, eight at 5 and 16, two batch tiles at 16), gate/up (448 groups) as a group-aligned
    stream-K grid of 224 CTAs holding two whole groups each, lm_head as stream-K with fix-ups."""
    cfg = OM.ModelConfig(n_layers=2, n_query_heads=16, n_kv_heads=4, head_dim=128, vocab_size=1000, max_seq_len=512,
                         mlp_hidden=14336)
    P = OM.random_params(cfg, 31, norm_jitter=0.1)
    _run(cfg, P, torch.bfloat16, n_seq=n_seq, t=96 if n_seq < 9 else 48, steps=2, seed=40 + n_seq, tol=1e-2)


def test_model_decode_deterministic_and_graph():
    """Two identical steps are bit-identical (stream-K partials summed in CTA order), and a
    CUDA-graph replay equals the eager step."""
    cfg = OM.ModelConfig(n_layers=2, n_query_heads=8, n_kv_heads=2, head_dim=128, vocab_size=1000, max_seq_len=512)
    P = OM.random_params(cfg, 14)
    seqs = _caches(cfg, _round(P, torch.bfloat16), 3, 100, 15)
    rc, _ = _ragged(cfg, seqs, torch.bfloat16, 4, 100)
    dm = M.DecodeModel(M.ModelConfig(n_layers=2, n_query_heads=8, n_kv_heads=2, head_dim=128, vocab_size=1000,
                                     max_seq_len=512), P)
    dm.bind(rc)
    toks = torch.tensor([1, 2, 3], dtype=torch.int32, device=DEV)
    lens, seen = rc.lens.clone(), rc.tokens_seen.clone()
    a = dm.step(toks).clone()
    rc.lens.copy_(lens)
    rc.tokens_seen.copy_(seen)
    b = dm.step(toks).clone()
    assert torch.equal(a, b)
    rc.lens.copy_(lens)
    rc.tokens_seen.copy_(seen)
    out = torch.empty_like(a)
    g = dm.capture(toks, out)
    g.replay()
    torch.cuda.synchronize()
    dm.ws.status()
    assert torch.equal(out, a)
    assert rc.tokens_seen.cpu().tolist() == [101] * 3


def test_model_decode_errors():
    """model.cpp:213-215: token id out of vocab / sequence exceeds max_seq_len -> contract_error."""
    cfg = OM.ModelConfig(n_layers=1, n_query_heads=4, n_kv_heads=2, head_dim=16, vocab_size=50, max_seq_len=60)
    P = OM.random_params(cfg, 16)
    seqs = _caches(cfg, P, 1, 59, 17)
    rc, _ = _ragged(cfg, seqs, torch.float32, 4, 59)
    dm = M.DecodeModel(M.ModelConfig(n_layers=1, n_query_heads=4, n_kv_heads=2, head_dim=16, vocab_size=50,
                                     max_seq_len=60), P, dtype=torch.float32)
    dm.bind(rc)
    with pytest.raises(lkv.ContractError):
        dm.step(torch.tensor([50], dtype=torch.int32, device=DEV))
    rc.tokens_seen.fill_(60)
    with pytest.raises(lkv.ContractError):
        dm.step(torch.tensor([3], dtype=torch.int32, device=DEV))
    with pytest.raises(lkv.UnsupportedError):  # bf16 needs head_dim 128
        M.DecodeModel(M.ModelConfig(n_layers=1, n_query_heads=4, n_kv_heads=2, head_dim=16, vocab_size=50), P)


@pytest.mark.skipif(O.ref_lib() is None, reason="oracle/_ref not built")
def test_model_decode_vs_reference_decode_step():
    """The reference's own init_model weights and decode_step (model.cpp, compiled in oracle/_ref)."""
    cfg = OM.ModelConfig(n_layers=2, n_query_heads=8, n_kv_heads=2, head_dim=16, vocab_size=128, max_seq_len=64)
    R = OM.RefModel(cfg)
    P = _round(R.params(), torch.float32)
    R.set_params(P)
    seqs = _caches(cfg, P, 1, 30, 18)
    rc, heads = _ragged(cfg, seqs, torch.float32, 3, 30)
    dm = M.DecodeModel(M.ModelConfig(n_layers=2, n_query_heads=8, n_kv_heads=2, head_dim=16, vocab_size=128,
                                     max_seq_len=64), P, dtype=torch.float32)
    dm.bind(rc)
    toks = [5, 77]
    lref, nk, _, ts = R.decode_steps(heads[0], 30, toks)
    for s, tk in enumerate(toks):
        lg = dm.step(torch.tensor([tk], dtype=torch.int32, device=DEV)).cpu().numpy()[0]
        assert rel_gap(lg, lref[s]) <= 1e-5
    assert ts == int(rc.tokens_seen[0]) == 32
