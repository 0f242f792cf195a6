"""Head-sharded eviction + decode over several GPUs (one process per GPU).

A rank owns a contiguous layer range [l0, l1) of every sequence (shard.layer_ranges), i.e. the
flat per-sequence heads [l0*H, l1*H).  Everything on the data path is local to the rank:
scoring, top-k, compaction and decode of its heads (lkv_evict_shard / lkv_decode_step).  The
path's only exchanges go through the library's NCCL communicator (lkv_comm_*):

* LKV-H logits: each rank contributes its heads' logits; one allgatherv gives every rank the
  full vector, and every rank solves the global Soft-TopK threshold (policy.cpp:110-120)
  redundantly and bit-identically inside lkv_evict_shard -- no budget exchange is needed.
* decode outputs: each rank's [n_seq][l1-l0][Hq][D] block is gathered to the root (gatherv),
  batched over the layers of one step, and reassembled to [n_seq][L][Hq][D].

`Comm` wraps lkv_comm_* (NCCL); `TorchComm` is the same interface over a torch.distributed
process group (gloo on CPU) so the host logic -- displacements, reassembly, budget agreement --
runs in world_size-2 CPU tests.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _abi
from . import shard as _shard
from . import (BUDGET_EXACT, ContractError, DenseCache, RaggedCache, Scorers, Workspace, _check, _ptr, _stream,
               decode_step, lib)


# ---- communicators ---------------------------------------------------------------------------------
class Comm:
    """lkv_comm_t (NCCL over NVLink/NVSwitch).  The unique id travels over the default
    torch.distributed group (any backend); the collectives themselves are the library's."""

    def __init__(self, world: int, rank: int, uid: bytes):
        if len(uid) != _abi.COMM_ID_BYTES:
            raise ContractError("NCCL unique id must be 128 bytes")
        self.world, self.rank = int(world), int(rank)
        self._h = C.c_void_p()
        buf = C.create_string_buffer(uid, _abi.COMM_ID_BYTES)
        _check(lib().lkv_comm_init(C.byref(self._h), buf, self.world, self.rank))

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(_abi.COMM_ID_BYTES)
        _check(lib().lkv_comm_get_unique_id(buf))
        return buf.raw

    @classmethod
    def from_process_group(cls) -> "Comm":
        import torch.distributed as dist

        if not dist.is_initialized():
            return cls(1, 0, cls.unique_id())
        obj = [cls.unique_id() if dist.get_rank() == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return cls(dist.get_world_size(), dist.get_rank(), obj[0])

    def close(self):
        if self._h:
            _check(lib().lkv_comm_destroy(self._h))
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def _tables(counts, displs):
        n = len(counts)
        return (C.c_int64 * n)(*[int(x) for x in counts]), (C.c_int64 * n)(*[int(x) for x in displs])

    def allgatherv(self, send: torch.Tensor, recv: torch.Tensor, counts, displs, stream=None) -> None:
        """recv[displs[r]: displs[r] + counts[r]] <- rank r's send (element units of recv)."""
        es = recv.element_size()
        b, d = self._tables([c * es for c in counts], [x * es for x in displs])
        _check(lib().lkv_comm_allgatherv(self._h, _ptr(send), _ptr(recv), b, d, _stream(stream)))

    def gatherv(self, send: torch.Tensor, recv: torch.Tensor | None, counts, displs, root: int = 0,
                stream=None) -> None:
        es = send.element_size()
        b, d = self._tables([c * es for c in counts], [x * es for x in displs])
        _check(lib().lkv_comm_gatherv(self._h, _ptr(send), _ptr(recv), b, d, int(root), _stream(stream)))


class TorchComm:
    """The Comm interface over torch.distributed (gloo/nccl) -- CPU tests of the host logic."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist, self.group = dist, group
        self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)

    def close(self):
        pass

    def allgatherv(self, send, recv, counts, displs, stream=None):
        m = max(int(c) for c in counts)
        # gloo exchanges host tensors: device data is staged through the host
        host = self.dist.get_backend(self.group) == "gloo"
        pad = torch.zeros(m, dtype=recv.dtype, device="cpu" if host else recv.device)
        pad[: int(counts[self.rank])] = send.reshape(-1)[: int(counts[self.rank])].to(pad.device)
        parts = [torch.zeros_like(pad) for _ in range(self.world)]
        self.dist.all_gather(parts, pad, group=self.group)
        flat = recv.view(-1)
        for r in range(self.world):
            flat[int(displs[r]): int(displs[r]) + int(counts[r])] = parts[r][: int(counts[r])].to(flat.device)

    def gatherv(self, send, recv, counts, displs, root=0, stream=None):
        tmp = torch.empty(int(sum(int(c) for c in counts)), dtype=send.dtype, device=send.device)
        self.allgatherv(send, tmp, counts, [sum(int(c) for c in counts[:r]) for r in range(self.world)])
        if self.rank == root:
            flat = recv.view(-1)
            off = 0
            for r in range(self.world):
                flat[int(displs[r]): int(displs[r]) + int(counts[r])] = tmp[off: off + int(counts[r])]
                off += int(counts[r])


# ---- shard plan ------------------------------------------------------------------------------------------
class ShardPlan:
    """Head shards of an L x H cache over `world` ranks: contiguous layer ranges (default), or --
    with per-head `weights` (e.g. eviction bytes t * in_bytes + budget * gather bytes, known before
    eviction because budgets depend only on the logits) -- a deterministic LPT assignment
    (shard.lpt_assign) that balances the skewed LKV-H budgets across ranks.  heads[r] is the sorted
    list of global flat heads l * H + h that rank r owns."""

    def __init__(self, n_layers: int, n_kv_heads: int, world: int, weights=None):
        self.n_layers, self.n_kv_heads, self.world = n_layers, n_kv_heads, world
        self.layers = _shard.layer_ranges(n_layers, world)
        self.lpt = weights is not None
        if self.lpt:
            if len(weights) != n_layers * n_kv_heads:
                raise ContractError("one LPT weight per (layer, kv head)")
            owner = _shard.lpt_assign(list(weights), world)
            self.heads = [[i for i, o in enumerate(owner) if o == r] for r in range(world)]
            self.imbalance = _shard.imbalance(list(weights), owner, world)
        else:
            self.heads = [list(range(l0 * n_kv_heads, l1 * n_kv_heads)) for l0, l1 in self.layers]
            owner = [r for r, hs in enumerate(self.heads) for _ in hs]
            self.imbalance = _shard.imbalance(list(weights), owner, world) if weights is not None else None

    def head_range(self, rank: int):
        if self.lpt:
            raise ContractError("an LPT plan owns a head list, not a range (heads[rank])")
        l0, l1 = self.layers[rank]
        return l0 * self.n_kv_heads, (l1 - l0) * self.n_kv_heads

    def n_local(self, rank: int) -> int:
        return len(self.heads[rank])

    def logit_counts(self):
        """Element counts / displacements of the rank-major logits buffer (global order for a
        layer-range plan; the LPT plan scatters it with `order`)."""
        counts = [len(h) for h in self.heads]
        return counts, [sum(counts[:r]) for r in range(self.world)]

    def order(self) -> list:
        """Global flat head of every position of the rank-major buffer."""
        return [h for hs in self.heads for h in hs]

    def order_tensor(self, device):
        key = str(device)
        if getattr(self, "_order_t", None) is None or self._order_key != key:
            self._order_t, self._order_key = torch.tensor(self.order(), device=device), key
        return self._order_t

    def output_counts(self, n_seq: int, per_layer: int):
        """Element counts/displacements of the rank-major gather buffer of decode outputs
        (per_layer = elements per layer of one sequence, Hq * D; a rank's block is its heads' share)."""
        per_head = per_layer // self.n_kv_heads
        counts = [n_seq * len(hs) * per_head for hs in self.heads]
        displs = [sum(counts[:r]) for r in range(self.world)]
        return counts, displs

    def assemble(self, gathered: torch.Tensor, n_seq: int, Hq: int, D: int) -> torch.Tensor:
        """Rank-major [r][n_seq][heads of r][G][D] blocks -> [n_seq][L][Hq][D]."""
        counts, displs = self.output_counts(n_seq, Hq * D)
        G = Hq // self.n_kv_heads
        blocks = [gathered.view(-1)[displs[r]: displs[r] + counts[r]].view(n_seq, -1, G, D) for r in range(self.world)]
        rank_major = torch.cat(blocks, dim=1)  # [n_seq][L*H in rank-major head order][G][D]
        out = torch.empty_like(rank_major)
        out[:, torch.tensor(self.order(), device=rank_major.device)] = rank_major
        return out.view(n_seq, self.n_layers, Hq, D)


def gather_logits(comm, plan: ShardPlan, local_logits: torch.Tensor) -> torch.Tensor:
    """Every rank's heads' LKV-H logits -> the full [L*H] vector on every rank."""
    counts, displs = plan.logit_counts()
    if local_logits.numel() != counts[comm.rank]:
        raise ContractError("local logits must cover exactly this rank's heads")
    out = torch.empty(plan.n_layers * plan.n_kv_heads, dtype=torch.float64, device=local_logits.device)
    comm.allgatherv(local_logits.to(torch.float64).contiguous(), out, counts, displs)
    if plan.lpt:  # rank-major -> global head order
        full = torch.empty_like(out)
        full[plan.order_tensor(out.device)] = out
        return full
    return out


# ---- the per-rank eviction -------------------------------------------------------------------------------
class ShardEvictor:
    """lkv_evict_shard on this rank's layer range of a dense cache (buffers allocated once).
    `cache` / `scorers` hold ONLY the local layers; budgets come from the global logits."""

    def __init__(self, cache: DenseCache, scorers: Scorers, plan: ShardPlan, rank: int, target_ratio: float,
                 mode: int = BUDGET_EXACT, decode_slack: int = 0, keep_scores: bool = False):
        """Layer-range plan: `cache` / `scorers` hold this rank's layers.  LPT plan: `cache` holds the
        rank's heads in plan.heads[rank] order, grouped any way as [n_seq][g][n_local / g][T][D] (the
        grouping only sets the host path's upload chunks), with one scorer per local head (scorer of
        local flat head j = j)."""
        n_seq, L, H, T, D = cache.shape
        n_local = plan.n_local(rank)
        if plan.lpt:
            if L * H != n_local:
                raise ContractError("an LPT shard's cache holds exactly its n_local heads")
            self.head_begin = 0
            self.head_ids = torch.tensor(plan.heads[rank], dtype=torch.int32, device=cache.keys.device)
        else:
            self.head_begin = plan.head_range(rank)[0]
            self.head_ids = None
            if L * H != n_local or H != plan.n_kv_heads:
                raise ContractError("local cache must hold exactly this rank's layer range")
        self.cache, self.scorers, self.plan = cache, scorers, plan
        self.n_logits = plan.n_layers * plan.n_kv_heads
        self.R, self.mode = float(target_ratio), mode
        cd = cache.desc()
        cap = lib().lkv_ragged_capacity_shard(C.byref(cd), self.n_logits, self.R, decode_slack)
        if cap < 0:
            _check(_abi.CONTRACT)
        dev = cache.keys.device
        self.ragged = RaggedCache(n_seq, L, H, D, cache.keys.dtype, cap, decode_slack, device=dev)
        nbytes = lib().lkv_workspace_bytes(C.byref(cd), self.n_logits)
        self.ws = Workspace(nbytes, device=dev)
        self.scores = torch.zeros(n_seq, L, H, T, dtype=torch.float32, device=dev) if keep_scores else None
        self.ratios = torch.empty(self.n_logits, dtype=torch.float64, device=dev)
        self.budgets = torch.empty(n_seq, n_local, dtype=torch.int32, device=dev)
        self._cd, self._sd, self._rd = cd, scorers.desc(), self.ragged.desc()

    def launch(self, logits: torch.Tensor, stream=None) -> None:
        if logits.numel() != self.n_logits or logits.dtype != torch.float64:
            raise ContractError("evict_shard needs the full fp64 logit vector (gather_logits)")
        if self.head_ids is not None:
            _check(lib().lkv_evict_heads(C.byref(self._cd), C.byref(self._sd), _ptr(logits), self.n_logits,
                                         _ptr(self.head_ids), self.R, self.mode, C.byref(self._rd), _ptr(self.scores),
                                         _ptr(self.ratios), _ptr(self.budgets), C.c_void_p(self.ws.ptr),
                                         self.ws.nbytes, _stream(stream)))
            return
        _check(lib().lkv_evict_shard(C.byref(self._cd), C.byref(self._sd), _ptr(logits), self.n_logits,
                                     self.head_begin, self.R, self.mode, C.byref(self._rd), _ptr(self.scores),
                                     _ptr(self.ratios), _ptr(self.budgets), C.c_void_p(self.ws.ptr), self.ws.nbytes,
                                     _stream(stream)))

    def launch_host(self, logits: torch.Tensor, host_keys: torch.Tensor, host_values: torch.Tensor,
                    host_out: RaggedCache | None = None, layers_per_chunk: int = 1, stream=None) -> None:
        """lkv_evict_host_shard: this rank's layers held in pinned host memory, K streamed into the
        evictor's device K buffer chunk by chunk, kept V rows gathered over PCIe, the compacted shard
        copied back into `host_out` (pinned, same capacity) when given."""
        if logits.numel() != self.n_logits or logits.dtype != torch.float64:
            raise ContractError("evict_host_shard needs the full fp64 logit vector (gather_logits)")
        if not (host_keys.is_pinned() and host_values.is_pinned()):
            raise ContractError("host K/V must be pinned (torch pin_memory)")
        if tuple(host_keys.shape) != self.cache.shape or host_keys.dtype != self.cache.keys.dtype:
            raise ContractError("host K/V must match the shard's cache shape and dtype")
        hd = _abi.CacheDesc(*[getattr(self._cd, f) for f, _ in _abi.CacheDesc._fields_])
        hd.keys, hd.values = host_keys.data_ptr(), host_values.data_ptr()
        dev_v = self.cache.values.data_ptr() if self.scorers.input == _abi.SCORER_KV else None
        ho = host_out.desc() if host_out is not None else None
        if self.head_ids is not None:
            _check(lib().lkv_evict_host_heads(C.byref(hd), C.c_void_p(self.cache.keys.data_ptr()),
                                              C.c_void_p(dev_v) if dev_v else None, C.byref(self._sd), _ptr(logits),
                                              self.n_logits, _ptr(self.head_ids), self.R, self.mode, C.byref(self._rd),
                                              C.byref(ho) if ho is not None else None, layers_per_chunk,
                                              C.c_void_p(self.ws.ptr), self.ws.nbytes, _stream(stream)))
            return
        _check(lib().lkv_evict_host_shard(C.byref(hd), C.c_void_p(self.cache.keys.data_ptr()),
                                          C.c_void_p(dev_v) if dev_v else None, C.byref(self._sd), _ptr(logits),
                                          self.n_logits, self.head_begin, self.R, self.mode, C.byref(self._rd),
                                          C.byref(ho) if ho is not None else None, layers_per_chunk,
                                          C.c_void_p(self.ws.ptr), self.ws.nbytes, _stream(stream)))

    def host_result_buffer(self) -> RaggedCache:
        r = self.ragged
        return RaggedCache(r.n_seq, r.n_layers, r.n_kv_heads, r.head_dim, r.dtype, r.capacity_rows, r.decode_slack,
                           device="cpu", pinned=True)

    def run(self, logits: torch.Tensor) -> RaggedCache:
        self.launch(logits)
        self.ws.status()
        self.ragged.tokens_seen.copy_(torch.tensor(self.cache.seq_lens, dtype=torch.int32))
        return self.ragged


def decode_and_gather(comm, plan: ShardPlan, ragged: RaggedCache, q, new_k, new_v, out_local=None,
                      gathered=None, root: int = 0, check: bool = False):
    """One decode step on this rank's layers, then the outputs gathered to `root`.
    Returns the rank-major gather buffer on root (plan.assemble() orders it), else None."""
    n_seq, Lr, Hq, D = q.shape
    out_local = decode_step(ragged, q, new_k, new_v, out=out_local, check=check)
    G = Hq // ragged.n_kv_heads
    counts, displs = plan.output_counts(n_seq, G * plan.n_kv_heads * D)
    if comm.rank == root and gathered is None:
        gathered = torch.empty(sum(counts), dtype=q.dtype, device=q.device)
    comm.gatherv(out_local.reshape(-1), gathered if comm.rank == root else None, counts, displs, root)
    return gathered if comm.rank == root else None
