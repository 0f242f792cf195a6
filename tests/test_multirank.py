"""Multi-rank host logic on CPU with the gloo backend (world_size 2): the GPU path shards
with no data-path collective, so what must hold across ranks is (i) identical LKV-H budgets
computed redundantly from the same logits, (ii) a disjoint, complete partition of the heads,
and (iii) the max-over-ranks timing reduction."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2605_06676_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # (i) redundant LKV-H solve: same logits -> bit-identical budgets on every rank
        rng = np.random.default_rng(1005)
        logits = rng.normal(0, 1.5, 640)
        b = O.freeze_budgets_exact(O.allocate_budgets(logits, 0.10), 0.10, 65536)
        mine = torch.tensor(b, dtype=torch.int64)
        gathered = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(gathered, mine)
        assert all(torch.equal(g, gathered[0]) for g in gathered)
        # (ii) partitions agree and cover everything exactly once
        ranges = shard.layer_ranges(80, world)
        l0, l1 = ranges[rank]
        owned = torch.zeros(80, dtype=torch.int64)
        owned[l0:l1] = 1
        dist.all_reduce(owned)
        assert torch.equal(owned, torch.ones(80, dtype=torch.int64))
        owner = shard.lpt_assign([int(x) for x in b], world)
        cnt = torch.tensor([sum(int(x) for x, o in zip(b, owner) if o == rank)], dtype=torch.int64)
        dist.all_reduce(cnt)
        assert int(cnt.item()) == int(np.sum(b))
        # (iii) timing = max over ranks
        t = shard.max_over_ranks(1.0 + rank)
        assert t == float(world)
        with open(os.path.join(out_dir, f"ok{rank}"), "w") as f:
            f.write("ok")
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    assert all((tmp_path / f"ok{r}").exists() for r in range(world))


def test_layer_ranges_and_batch_shard():
    for L in (1, 32, 80):
        for W in (1, 2, 4, 8):
            rs = shard.layer_ranges(L, W)
            assert rs[0][0] == 0 and rs[-1][1] == L
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1
    owned = sorted(s for r in range(4) for s in shard.batch_shard(16, 4, r))
    assert owned == list(range(16))
    with pytest.raises(ValueError):
        shard.batch_shard(4, 2, 2)


def test_lpt_balances_skewed_budgets():
    rng = np.random.default_rng(5)
    logits = rng.normal(0, 1.5, 640)  # C5's skewed LKV-H logits
    b = O.freeze_budgets_exact(O.allocate_budgets(logits, 0.10), 0.10, 65536)
    owner = shard.lpt_assign([int(x) for x in b], 8)
    assert sorted(set(owner)) == list(range(8))
    assert shard.imbalance([int(x) for x in b], owner, 8) < 1.01
    # contiguous ranges are far worse for decode on skewed budgets: LPT is what fixes it
    contiguous = [min(i * 8 // 640, 7) for i in range(640)]
    assert shard.imbalance([int(x) for x in b], contiguous, 8) > shard.imbalance([int(x) for x in b], owner, 8)
    # deterministic
    assert owner == shard.lpt_assign([int(x) for x in b], 8)


def _sharded_worker(rank, world, port, out_dir):
    """The head-sharded path's host logic through the same interface the NCCL communicator
    implements (sharded.TorchComm over gloo): logits allgatherv, decode-output gatherv and
    reassembly, budgets agreeing on every rank."""
    from paper_2605_06676_b200 import sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = sharded.TorchComm()
        L, H, Hq, D, n_seq = 5, 8, 32, 16, 3  # 5 layers over 2 ranks: uneven ranges (3 + 2)
        plan = sharded.ShardPlan(L, H, world)
        rng = np.random.default_rng(77)
        full = torch.tensor(rng.normal(0, 1, L * H))
        h0, n = plan.head_range(rank)
        got = sharded.gather_logits(comm, plan, full[h0:h0 + n].clone())
        assert torch.equal(got, full)  # every rank holds the full logit vector
        # every rank's redundant solve agrees; its slice is its heads' budgets
        b = O.freeze_budgets_exact(O.allocate_budgets(got.numpy(), 0.15), 0.15, 4096)
        mine = torch.tensor(b[h0:h0 + n], dtype=torch.int64)
        parts = [torch.zeros(plan.head_range(r)[1], dtype=torch.int64) for r in range(world)]
        padded = [torch.zeros(L * H, dtype=torch.int64) for _ in range(world)]
        pad = torch.zeros(L * H, dtype=torch.int64)
        pad[:n] = mine
        dist.all_gather(padded, pad)
        for r in range(world):
            parts[r] = padded[r][: plan.head_range(r)[1]]
        assert torch.equal(torch.cat(parts), torch.tensor(b, dtype=torch.int64))
        assert int(torch.cat(parts).sum()) == round(0.15 * L * H * 4096)
        # decode outputs: element (s, l, qh, d) encodes its global coordinates
        l0, l1 = plan.layers[rank]
        s_i, l_i, q_i, d_i = torch.meshgrid(torch.arange(n_seq), torch.arange(l0, l1), torch.arange(Hq),
                                            torch.arange(D), indexing="ij")
        local = (((s_i * 100 + l_i) * 100 + q_i) * 100 + d_i).to(torch.float64)
        counts, displs = plan.output_counts(n_seq, Hq * D)
        gathered = torch.empty(sum(counts), dtype=torch.float64) if rank == 0 else None
        comm.gatherv(local.reshape(-1), gathered, counts, displs, root=0)
        if rank == 0:
            out = plan.assemble(gathered, n_seq, Hq, D)
            s_i, l_i, q_i, d_i = torch.meshgrid(torch.arange(n_seq), torch.arange(L), torch.arange(Hq),
                                                torch.arange(D), indexing="ij")
            assert torch.equal(out, (((s_i * 100 + l_i) * 100 + q_i) * 100 + d_i).to(torch.float64))
        with open(os.path.join(out_dir, f"ok{rank}"), "w") as f:
            f.write("ok")
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_head_sharded_host_logic(tmp_path):
    world = 2
    mp.spawn(_sharded_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    assert all((tmp_path / f"ok{r}").exists() for r in range(world))


def test_shard_plan_ranges():
    from paper_2605_06676_b200 import sharded

    for L, W in ((32, 8), (80, 8), (5, 2), (3, 4)):
        plan = sharded.ShardPlan(L, 8, W)
        counts, displs = plan.logit_counts()
        assert sum(counts) == L * 8 and displs[0] == 0
        assert all(displs[r] + counts[r] == displs[r + 1] for r in range(W - 1))


def _lpt_worker(rank, world, port, out_dir):
    """The LPT head placement's host logic (sharded.ShardPlan with weights) over gloo: every rank
    derives the same plan, the rank-major logits allgatherv is scattered back to global order, and
    the decode outputs of arbitrary head lists reassemble into [n_seq][L][Hq][D]."""
    from paper_2605_06676_b200 import sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = sharded.TorchComm()
        L, H, G, D, n_seq, T = 6, 4, 2, 8, 2, 4096
        rng = np.random.default_rng(91)
        full = torch.tensor(rng.normal(0, 1.5, L * H))
        b = O.freeze_budgets_exact(O.allocate_budgets(full.numpy(), 0.1), 0.1, T)
        plan = sharded.ShardPlan(L, H, world, weights=[T * 264 + int(x) * 1028 for x in b])
        assert plan.lpt and sorted(h for hs in plan.heads for h in hs) == list(range(L * H))
        assert plan.imbalance < 1.05  # 24 heads over 2 ranks: LPT granularity
        mine = plan.heads[rank]
        got = sharded.gather_logits(comm, plan, full[mine].clone())
        assert torch.equal(got, full)
        # outputs: rank r holds [n_seq][1][n_local * G][D] for its heads, in plan order
        s_i, j_i, g_i, d_i = torch.meshgrid(torch.arange(n_seq), torch.tensor(mine), torch.arange(G), torch.arange(D),
                                            indexing="ij")
        local = (((s_i * 100 + j_i) * 10 + g_i) * 100 + d_i).to(torch.float64).reshape(n_seq, 1, len(mine) * G, D)
        counts, displs = plan.output_counts(n_seq, G * H * D)
        gathered = torch.empty(sum(counts), dtype=torch.float64) if rank == 0 else None
        comm.gatherv(local.reshape(-1), gathered, counts, displs, root=0)
        if rank == 0:
            out = plan.assemble(gathered, n_seq, H * G, D)
            s_i, l_i, q_i, d_i = torch.meshgrid(torch.arange(n_seq), torch.arange(L), torch.arange(H * G),
                                                torch.arange(D), indexing="ij")
            flat = l_i * H + q_i // G
            assert torch.equal(out, (((s_i * 100 + flat) * 10 + q_i % G) * 100 + d_i).to(torch.float64))
        with open(os.path.join(out_dir, f"ok{rank}"), "w") as f:
            f.write("ok")
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_lpt_placement(tmp_path):
    world = 2
    mp.spawn(_lpt_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    assert all((tmp_path / f"ok{r}").exists() for r in range(world))
