"""Head-sharded eviction + decode on one B200.

Every shard is independent on the data path, so the N-rank result can be checked on one GPU by
running each rank's shard in turn (no kernel waits on another rank) and comparing the union with
the unsharded path: budgets, offsets, kept positions and rows bit-exact, decode outputs equal.
The NCCL communicator (lkv_comm_*) is exercised with a 1-rank communicator: allgatherv and
gatherv through NCCL on this GPU.
"""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2605_06676_b200 as lkv
from paper_2605_06676_b200 import sharded, synth

pytestmark = pytest.mark.gpu


def _local(cache, scorers, l0, l1):
    c = lkv.DenseCache(cache.keys[:, l0:l1].contiguous(), cache.values[:, l0:l1].contiguous(), cache.seq_lens)
    s = lkv.Scorers(scorers.w1[l0:l1], scorers.b1[l0:l1], scorers.w2[l0:l1], input=scorers.input,
                    activation=scorers.activation, stride_layer=1, stride_head=0)
    return c, s


@pytest.mark.parametrize("cid,world,L,T", [(2, 4, 8, 5000), (2, 3, 8, 4096), (4, 2, 5, 6000), (5, 8, 8, 3000)])
def test_head_shards_equal_unsharded(cid, world, L, T):
    cfg = synth.CONFIGS[cid]
    S = min(cfg.n_seq, 3)
    cache = synth.make_cache(cfg, n_layers=L, max_tokens=T, n_seq=S)
    scorers = synth.make_scorers(cfg, n_layers=L)
    logits = synth.make_logits(cfg, n_layers=L)
    full = lkv.evict(cache, scorers, logits, cfg.ratio, lkv.BUDGET_EXACT, decode_slack=4, keep_scores=False)
    H = cfg.n_kv_heads
    plan = sharded.ShardPlan(L, H, world)
    # the oracle's budgets from the same logits (K2 bit-exact on every rank)
    want_b = [O.freeze_budgets_exact(O.allocate_budgets(logits.cpu().numpy(), cfg.ratio), cfg.ratio, t)
              for t in cache.seq_lens]
    G = cfg.n_q_heads // H
    steps = [synth.make_decode_inputs(cfg, s, n_layers=L, n_seq=S) for s in range(3)]
    shard_out = [[] for _ in range(3)]
    for r in range(world):
        l0, l1 = plan.layers[r]
        if l1 == l0:
            continue
        lc, ls = _local(cache, scorers, l0, l1)
        ev = sharded.ShardEvictor(lc, ls, plan, r, cfg.ratio, lkv.BUDGET_EXACT, decode_slack=4)
        rc = ev.run(logits)
        h0, n = plan.head_range(r)
        for s in range(S):
            assert (ev.budgets[s].cpu().numpy() == want_b[s][h0:h0 + n]).all()
        assert torch.equal(rc.lens.view(S, -1), full.cache.lens.view(S, -1)[:, h0:h0 + n])
        for s in range(S):
            for j in range(n):
                k, v, p = rc.head(s * n + j)
                kf, vf, pf = full.cache.head(s * L * H + h0 + j)
                assert torch.equal(p, pf) and torch.equal(k, kf) and torch.equal(v, vf)
        for st in range(3):
            q, k, v = (x[:, l0:l1].contiguous() for x in steps[st])
            shard_out[st].append(lkv.decode_step(rc, q, k, v).clone())
    full_out = [lkv.decode_step(full.cache, *steps[s]).clone() for s in range(3)]  # after the layout checks
    for st in range(3):
        got = torch.cat(shard_out[st], dim=1)
        assert got.shape == full_out[st].shape
        assert torch.allclose(got.float(), full_out[st].float(), rtol=0, atol=1e-6 * float(full_out[st].float().abs().max()))


def test_evict_shard_contract_errors():
    cfg = synth.CONFIGS[2]
    cache = synth.make_cache(cfg, n_layers=4, max_tokens=1000)
    scorers = synth.make_scorers(cfg, n_layers=4)
    plan = sharded.ShardPlan(8, 8, 2)  # the 4 local layers are rank 1's layers 4..7
    ev = sharded.ShardEvictor(cache, scorers, plan, 1, 0.15)
    with pytest.raises(lkv.ContractError):
        ev.launch(synth.make_logits(cfg, n_layers=4))  # not the full logit vector
    with pytest.raises(lkv.ContractError):
        sharded.ShardEvictor(cache, scorers, sharded.ShardPlan(8, 8, 4), 1, 0.15)  # wrong layer count
    ev.run(synth.make_logits(cfg, n_layers=8))
    with pytest.raises(lkv.BudgetError):
        sharded.ShardEvictor(cache, scorers, plan, 1, 1.5).run(synth.make_logits(cfg, n_layers=8))


def test_nccl_comm_single_rank():
    comm = sharded.Comm(1, 0, sharded.Comm.unique_id())
    try:
        x = torch.arange(40, dtype=torch.float64, device="cuda")
        out = torch.full((50,), -1.0, dtype=torch.float64, device="cuda")
        comm.allgatherv(x, out, [40], [7])
        torch.cuda.synchronize()
        assert torch.equal(out[7:47], x) and (out[:7] == -1).all() and (out[47:] == -1).all()
        y = torch.randn(3, 5, 32, 16, device="cuda").to(torch.bfloat16)
        g = torch.zeros(y.numel() + 10, dtype=torch.bfloat16, device="cuda")
        comm.gatherv(y.reshape(-1), g, [y.numel()], [10], root=0)
        torch.cuda.synchronize()
        assert torch.equal(g[10:], y.reshape(-1))
        # the sharded helpers on a 1-rank communicator
        plan = sharded.ShardPlan(4, 8, 1)
        lg = torch.randn(32, dtype=torch.float64, device="cuda")
        assert torch.equal(sharded.gather_logits(comm, plan, lg), lg)
    finally:
        comm.close()


@pytest.mark.parametrize("world,rank", [(4, 1), (4, 3)])
def test_host_shard_equals_device_shard(world, rank):
    """lkv_evict_host_shard (the rank's layers in pinned host memory, K streamed in, kept V gathered
    over PCIe, compacted shard copied back) == lkv_evict_shard on the device copy, bit for bit."""
    cfg = synth.CONFIGS[2]
    L, T = 8, 5000
    cache = synth.make_cache(cfg, n_layers=L, max_tokens=T)
    scorers = synth.make_scorers(cfg, n_layers=L)
    logits = synth.make_logits(cfg, n_layers=L)
    plan = sharded.ShardPlan(L, cfg.n_kv_heads, world)
    l0, l1 = plan.layers[rank]
    lc, ls = _local(cache, scorers, l0, l1)
    ev = sharded.ShardEvictor(lc, ls, plan, rank, cfg.ratio, lkv.BUDGET_EXACT, decode_slack=2)
    dev = ev.run(logits)
    want = [x.clone() for x in (dev.offsets, dev.lens, dev.positions, dev.keys, dev.values)]
    hk, hv = lc.keys.cpu().pin_memory(), lc.values.cpu().pin_memory()
    ho = ev.host_result_buffer()
    for _ in range(2):
        ev.launch_host(logits, hk, hv, ho, layers_per_chunk=1)
        torch.cuda.synchronize()
        ev.ws.status()
        assert torch.equal(ho.offsets, want[0].cpu()) and torch.equal(ho.lens, want[1].cpu())
        offs, lens = want[0].cpu().tolist(), want[1].cpu().tolist()
        for h in range(len(lens)):
            o, n = offs[h], lens[h]
            assert torch.equal(ho.positions[o:o + n], want[2][o:o + n].cpu())
            assert torch.equal(ho.keys[o:o + n], want[3][o:o + n].cpu())
            assert torch.equal(ho.values[o:o + n], want[4][o:o + n].cpu())


def _lpt_local(cache, scorers, heads, H):
    """An LPT shard's inputs: its heads (any layers) as a [n_seq][1][n_local][T][D] cache with one
    scorer per local head."""
    ls = torch.tensor([h // H for h in heads], device="cuda")
    hs = torch.tensor([h % H for h in heads], device="cuda")
    K = cache.keys[:, ls, hs].unsqueeze(1).contiguous()
    V = cache.values[:, ls, hs].unsqueeze(1).contiguous()
    s = lkv.Scorers(scorers.w1[ls], scorers.b1[ls], scorers.w2[ls], input=scorers.input,
                    activation=scorers.activation, stride_layer=0, stride_head=1)
    return lkv.DenseCache(K, V, cache.seq_lens), s, ls, hs


@pytest.mark.parametrize("cid,world,L,T", [(3, 8, 8, 3000), (5, 4, 10, 2000), (4, 3, 6, 4000)])
def test_lpt_shards_equal_unsharded(cid, world, L, T):
    """LPT head placement (budget-balanced head lists, lkv_evict_heads): every rank's shard run in
    turn on this GPU; the union equals the unsharded eviction bit for bit (budgets, kept rows,
    positions) and the decode outputs, reassembled by the plan, equal the unsharded decode."""
    cfg = synth.CONFIGS[cid]
    S = min(cfg.n_seq, 2)
    cache = synth.make_cache(cfg, n_layers=L, max_tokens=T, n_seq=S)
    scorers = synth.make_scorers(cfg, n_layers=L)
    logits = synth.make_logits(cfg, n_layers=L)
    H = cfg.n_kv_heads
    full = lkv.evict(cache, scorers, logits, cfg.ratio, lkv.BUDGET_EXACT, decode_slack=4, keep_scores=False)
    b = O.freeze_budgets_exact(O.allocate_budgets(logits.cpu().numpy(), cfg.ratio), cfg.ratio, T)
    plan = sharded.ShardPlan(L, H, world, weights=[T * 264 + int(x) * 1028 for x in b])
    assert plan.lpt and plan.imbalance < 1.05
    G = cfg.n_q_heads // H
    steps = [synth.make_decode_inputs(cfg, s, n_layers=L, n_seq=S) for s in range(2)]
    got = [torch.zeros_like(steps[0][0]) for _ in range(2)]
    for r in range(world):
        heads = plan.heads[r]
        lc, ls_, ls, hs = _lpt_local(cache, scorers, heads, H)
        ev = sharded.ShardEvictor(lc, ls_, plan, r, cfg.ratio, lkv.BUDGET_EXACT, decode_slack=4)
        rc = ev.run(logits)
        n = len(heads)
        for s in range(S):
            assert (ev.budgets[s].cpu().numpy() == b[heads]).all()
            for j, hg in enumerate(heads):
                k, v, p = rc.head(s * n + j)
                kf, vf, pf = full.cache.head(s * L * H + hg)
                assert torch.equal(p, pf) and torch.equal(k, kf) and torch.equal(v, vf)
        for st in range(2):
            q, nk, nv = steps[st]
            qg = q.view(S, L, H, G, -1)[:, ls, hs].reshape(S, 1, n * G, -1).contiguous()
            out = lkv.decode_step(rc, qg, nk[:, ls, hs].unsqueeze(1).contiguous(), nv[:, ls, hs].unsqueeze(1).contiguous())
            got[st].view(S, L, H, G, -1)[:, ls, hs] = out.view(S, n, G, -1)
    for st in range(2):
        want = lkv.decode_step(full.cache, *steps[st])
        assert torch.allclose(got[st].float(), want.float(), rtol=0, atol=1e-6 * float(want.float().abs().max()))
