"""B200-native LKV inference-time eviction path (arxiv 2605.06676), Python harness side.

The product is ``liblkv_b200.so`` (sm_100a kernels behind the C ABI in
``include/lkv_b200.h``) and its C++ host layer; this package drives that ABI
with torch device buffers, mirroring the reference's hot-path API names
(``/root/reference/proj/include/lkv``):

=========================  ==============================================================
reference (C++, fp64)       here (device, via the C ABI)
=========================  ==============================================================
allocate_budgets            :func:`allocate_budgets`   (policy.hpp:67)
freeze_budgets              :func:`freeze_budgets`     (policy.hpp:70; + exact-sum mode)
token_scores                :func:`token_scores`       (policy.hpp:73)
inference_select/hard_topk  :func:`inference_select`   (policy.hpp:81, soft_topk.hpp:71)
cache_from_trace            :func:`cache_from_trace`   (model.hpp:99)
prefill_with_eviction       :func:`prefill_with_eviction` (evictsim.hpp:74, K/V-given form)
decode_step (attention)     :func:`decode_step`        (model.hpp:95)
kv_memory_bytes             :func:`kv_memory_bytes`    (evictsim.hpp:38-40)
=========================  ==============================================================

Errors raise the reference's exception taxonomy (``errors.hpp:10-32``).
There is no CPU fallback: every compute call launches CUDA kernels or raises.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import torch

from . import _abi
from ._abi import (BF16, BUDGET_EXACT, BUDGET_FLOOR, F32, GELU_ERF, SCORER_K, SCORER_KV, SILU,  # noqa: F401
                   CacheDesc, RaggedDesc, ScorerDesc)

__all__ = [
    "LkvError", "ContractError", "NumericError", "BudgetError", "OverflowGuardError", "DegenerateMaskError",
    "CudaError", "UnsupportedError", "DenseCache", "Scorers", "RaggedCache", "Workspace", "allocate_budgets",
    "freeze_budgets", "budgets", "token_scores", "inference_select", "select", "compact", "cache_from_trace",
    "evict", "prefill_with_eviction", "decode_plan", "decode_step", "kv_memory_bytes", "lib",
]


# ---- errors (errors.hpp:10-32) ---------------------------------------------------------------
class LkvError(RuntimeError):
    code = -1


class ContractError(LkvError):
    code = _abi.CONTRACT


class NumericError(LkvError):
    code = _abi.NUMERIC


class BudgetError(LkvError):
    code = _abi.BUDGET


class OverflowGuardError(LkvError):
    code = _abi.OVERFLOW_GUARD


class DegenerateMaskError(LkvError):
    code = _abi.DEGENERATE_MASK


class CudaError(LkvError):
    code = _abi.CUDA


class UnsupportedError(LkvError):
    code = _abi.UNSUPPORTED


class NcclError(LkvError):
    code = _abi.NCCL


_ERR = {c.code: c for c in (ContractError, NumericError, BudgetError, OverflowGuardError, DegenerateMaskError,
                            CudaError, UnsupportedError, NcclError)}


def lib():
    return _abi.load()


def _check(rc: int) -> None:
    if rc != 0:
        msg = lib().lkv_last_error().decode()
        raise _ERR.get(rc, LkvError)(msg)


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _dtype_code(dt: torch.dtype) -> int:
    if dt == torch.bfloat16:
        return BF16
    if dt == torch.float32:
        return F32
    raise ContractError(f"unsupported dtype {dt} (bf16 or fp32)")


# ---- containers --------------------------------------------------------------------------------
class Workspace:
    """Caller-owned device scratch (256-byte aligned) with the device error latch."""

    def __init__(self, nbytes: int, device="cuda"):
        self.nbytes = int(max(nbytes, 256))
        self._buf = torch.empty(self.nbytes + 256, dtype=torch.uint8, device=device)
        base = self._buf.data_ptr()
        self.ptr = (base + 255) & ~255
        _check(lib().lkv_workspace_init(C.c_void_p(self.ptr), self.nbytes, _stream()))

    def status(self, stream=None) -> None:
        """Synchronise and raise any device-side error latched since the last check."""
        _check(lib().lkv_workspace_status(C.c_void_p(self.ptr), _stream(stream)))


@dataclass
class DenseCache:
    """Pre-eviction K/V: [n_seq, n_layers, n_kv_heads, T, head_dim] (K post-RoPE, evictsim.cpp:143)."""

    keys: torch.Tensor
    values: torch.Tensor
    seq_lens: list

    def __post_init__(self):
        if self.keys.dim() != 5 or self.keys.shape != self.values.shape:
            raise ContractError("keys/values must be equal [n_seq, L, H, T, D] tensors")
        if self.keys.dtype != self.values.dtype:
            raise ContractError("keys/values dtype mismatch")
        self.keys = self.keys.contiguous()
        self.values = self.values.contiguous()
        n_seq, L, H, T, D = self.keys.shape
        self.seq_lens = [int(x) for x in (self.seq_lens if self.seq_lens is not None else [T] * n_seq)]
        self._lens_c = (C.c_int32 * max(len(self.seq_lens), 1))(*self.seq_lens)

    @property
    def shape(self):
        return tuple(self.keys.shape)

    @property
    def n_heads(self):
        n_seq, L, H, _, _ = self.keys.shape
        return n_seq * L * H

    def desc(self) -> CacheDesc:
        n_seq, L, H, T, D = self.keys.shape
        if len(self.seq_lens) != n_seq:
            raise ContractError("one sequence length per sequence required")
        return CacheDesc(n_seq, L, H, D, T, _dtype_code(self.keys.dtype), 0, self.keys.data_ptr(),
                         self.values.data_ptr(), C.cast(self._lens_c, C.POINTER(C.c_int32)))


@dataclass
class Scorers:
    """LKV-T scorers u = act(x W1 + b1) . w2 (policy.hpp:24-32).  w1 is [n_scorers, in, hidden]."""

    w1: torch.Tensor
    b1: torch.Tensor
    w2: torch.Tensor
    input: int = SCORER_K
    activation: int = GELU_ERF
    stride_layer: int = 1
    stride_head: int = 0

    def __post_init__(self):
        if self.w1.dim() != 3:
            raise ContractError("w1 must be [n_scorers, in, hidden]")
        self.w1t = self.w1.transpose(1, 2).contiguous()  # [n_scorers][hidden][in]: the K-major MMA operand
        self.b1 = self.b1.to(torch.float32).contiguous()
        self.w2 = self.w2.to(torch.float32).reshape(self.w1.shape[0], -1).contiguous()

    def desc(self) -> ScorerDesc:
        ns, _, hid = self.w1.shape
        return ScorerDesc(self.input, self.activation, hid, ns, self.stride_layer, self.stride_head,
                          self.w1t.data_ptr(), self.b1.data_ptr(), self.w2.data_ptr())


@dataclass
class RaggedCache:
    """Compacted per-head cache (KvCache/HeadCache, model.hpp:55-71) in one ragged buffer."""

    n_seq: int
    n_layers: int
    n_kv_heads: int
    head_dim: int
    dtype: torch.dtype
    capacity_rows: int
    decode_slack: int
    device: str = "cuda"
    pinned: bool = False
    offsets: torch.Tensor = field(init=False)
    lens: torch.Tensor = field(init=False)
    keys: torch.Tensor = field(init=False)
    values: torch.Tensor = field(init=False)
    positions: torch.Tensor = field(init=False)
    tokens_seen: torch.Tensor = field(init=False)

    def __post_init__(self):
        n = self.n_seq * self.n_layers * self.n_kv_heads
        kw = {"pin_memory": True} if self.pinned else {}
        self.offsets = torch.zeros(n + 1, dtype=torch.int64, device=self.device, **kw)
        self.lens = torch.zeros(n, dtype=torch.int32, device=self.device, **kw)
        rows = max(int(self.capacity_rows), 1)
        self.keys = torch.empty(rows, self.head_dim, dtype=self.dtype, device=self.device, **kw)
        self.values = torch.empty(rows, self.head_dim, dtype=self.dtype, device=self.device, **kw)
        self.positions = torch.full((rows,), -1, dtype=torch.int32, device=self.device, **kw)
        self.tokens_seen = torch.zeros(self.n_seq, dtype=torch.int32, device=self.device, **kw)
        self._decode_ws = None

    @property
    def n_heads(self):
        return self.n_seq * self.n_layers * self.n_kv_heads

    def desc(self) -> RaggedDesc:
        return RaggedDesc(self.n_heads, self.head_dim, _dtype_code(self.dtype), self.decode_slack,
                          int(self.capacity_rows), self.offsets.data_ptr(), self.lens.data_ptr(),
                          self.keys.data_ptr(), self.values.data_ptr(), self.positions.data_ptr())

    def head(self, i: int):
        """(keys, values, retained_positions) of flat head i (host sync)."""
        o = int(self.offsets[i])
        n = int(self.lens[i])
        return self.keys[o:o + n], self.values[o:o + n], self.positions[o:o + n]

    def retained(self):
        return self.lens.clone()


# ---- K2: budgets ----------------------------------------------------------------------------------
def budgets(logits: torch.Tensor, target_ratio: float, seq_lens, mode: int = BUDGET_FLOOR, decode_slack: int = 0,
            want_offsets: bool = False, ws: Workspace | None = None, check: bool = True):
    """LKV-H: ratios = soft_topk(logits, R*n, 1) then integer budgets per sequence length.
    Returns (ratios f64 [n], budgets i32 [n_seq, n][, offsets i64])."""
    logits = logits.to(torch.float64).contiguous()
    n = logits.numel()
    seq_lens = [int(t) for t in seq_lens]
    dev = logits.device
    ratios = torch.empty(n, dtype=torch.float64, device=dev)
    b = torch.empty(len(seq_lens), n, dtype=torch.int32, device=dev)
    offs = torch.empty(len(seq_lens) * n + 1, dtype=torch.int64, device=dev) if want_offsets else None
    ws = ws or Workspace(256, device=dev)
    lens_c = (C.c_int32 * max(len(seq_lens), 1))(*seq_lens)
    _check(lib().lkv_budgets(_ptr(logits), n, float(target_ratio), mode, lens_c, len(seq_lens), decode_slack,
                             _ptr(ratios), _ptr(b), _ptr(offs), C.c_void_p(ws.ptr), ws.nbytes, _stream()))
    if check:
        ws.status()
    return (ratios, b, offs) if want_offsets else (ratios, b)


def allocate_budgets(scores: torch.Tensor, target_ratio: float, n_layers: int, n_kv_heads: int) -> torch.Tensor:
    """policy.hpp:67 -- flat relaxed top-k over all head logits, k = R*L*H, tau = 1."""
    if not (0.0 < target_ratio < 1.0):
        raise BudgetError("target ratio must lie in (0,1)")
    if scores.dim() != 1 or scores.numel() != n_layers * n_kv_heads:
        raise ContractError("allocate_budgets: score length mismatch")
    ratios, _ = budgets(scores, target_ratio, [1])
    return ratios


def freeze_budgets(logits: torch.Tensor, target_ratio: float, t: int, exact: bool = False) -> torch.Tensor:
    """policy.hpp:70 -- floor(r * t) (or the exact-sum variant) straight from the logits."""
    if t < 1:
        raise ContractError("freeze_budgets: t must be >= 1")
    _, b = budgets(logits, target_ratio, [t], BUDGET_EXACT if exact else BUDGET_FLOOR)
    return b[0]


# ---- K1: scorer ------------------------------------------------------------------------------------
def token_scores(cache: DenseCache, scorers: Scorers, out: torch.Tensor | None = None, check: bool = True):
    """policy.hpp:73 for every (seq, layer, head) at once -> fp32 [n_seq, L, H, T]."""
    n_seq, L, H, T, D = cache.shape
    if out is None:
        out = torch.zeros(n_seq, L, H, T, dtype=torch.float32, device=cache.keys.device)
    cd, sd = cache.desc(), scorers.desc()
    _check(lib().lkv_score(C.byref(cd), C.byref(sd), _ptr(out), None, 0, _stream()))
    if check:
        torch.cuda.current_stream().synchronize()
    return out


# ---- K3/K4: select + compact ---------------------------------------------------------------------------
def _workspace_for(cache: DenseCache, n_logits: int) -> Workspace:
    cd = cache.desc()
    nbytes = lib().lkv_workspace_bytes(C.byref(cd), n_logits)
    if nbytes == 0:
        _check(_abi.CONTRACT)
    return Workspace(nbytes, device=cache.keys.device)


def _ragged_for(cache: DenseCache, rows: int, slack: int) -> RaggedCache:
    n_seq, L, H, T, D = cache.shape
    return RaggedCache(n_seq, L, H, D, cache.keys.dtype, rows, slack, device=cache.keys.device)


def select(cache: DenseCache, scores: torch.Tensor, budgets_: torch.Tensor, decode_slack: int = 0,
           gather: bool = True, ws: Workspace | None = None) -> RaggedCache:
    """Per-head top-b positions (ties -> lowest index), ascending; optionally gathers rows."""
    b = budgets_.to(torch.int32).reshape(-1).contiguous()
    if b.numel() != cache.n_heads:
        raise ContractError("one budget per head required")
    cap = int(b.clamp(min=0).sum().item()) + cache.n_heads * decode_slack
    rc = _ragged_for(cache, cap, decode_slack)
    _check(lib().lkv_ragged_offsets(_ptr(b), cache.n_heads, decode_slack, _ptr(rc.offsets), _stream()))
    ws = ws or _workspace_for(cache, 1)
    cd, rd = cache.desc(), rc.desc()
    scores = scores.contiguous()  # keep every temporary alive across the call (stream-ordered reuse)
    _check(lib().lkv_select(C.byref(cd), _ptr(scores), _ptr(b), C.byref(rd), 1 if gather else 0,
                            C.c_void_p(ws.ptr), ws.nbytes, _stream()))
    ws.status()
    rc.tokens_seen.copy_(torch.tensor(cache.seq_lens, dtype=torch.int32))
    return rc


def inference_select(scores: torch.Tensor, b: int) -> torch.Tensor:
    """policy.hpp:81 / soft_topk.hpp:71 -- int mask with exactly b ones at the largest scores."""
    t = scores.numel()
    if b < 0 or b > t:
        raise BudgetError("hard_topk: b outside [0, n]")
    sc = scores.to(torch.float32).reshape(1, 1, 1, t).contiguous()
    dummy = torch.zeros(1, 1, 1, t, 8, dtype=torch.float32, device=scores.device)
    cache = DenseCache(dummy, dummy, [t])
    rc = select(cache, sc, torch.tensor([b], dtype=torch.int32, device=scores.device), gather=False)
    mask = torch.zeros(t, dtype=torch.int32, device=scores.device)
    if b:
        mask[rc.positions[:b].long()] = 1
    return mask


hard_topk = inference_select


def compact(cache: DenseCache, ragged: RaggedCache, ws: Workspace | None = None) -> RaggedCache:
    """Gather rows positions[offsets[i] + r], r < lens[i], of every head (evictsim.cpp:202-215);
    a position outside [0, t) raises ContractError (nothing is written for that head)."""
    cd, rd = cache.desc(), ragged.desc()
    ws = ws or Workspace(256, device=cache.keys.device)
    _check(lib().lkv_compact(C.byref(cd), C.byref(rd), C.c_void_p(ws.ptr), ws.nbytes, _stream()))
    ws.status()
    return ragged


def cache_from_trace(cache: DenseCache, hard_masks: torch.Tensor, decode_slack: int = 0) -> RaggedCache:
    """model.hpp:99 -- keep the rows of each head whose binary mask is set (ascending).  The mask
    scan, ragged offsets and row gather run on the device (lkv_mask_counts, lkv_cache_from_trace);
    the host reads one number, the total, to allocate the ragged cache."""
    n_seq, L, H, T, D = cache.shape
    m = hard_masks.reshape(cache.n_heads, -1)
    if m.shape[1] != T and m.shape[1] != max(cache.seq_lens):
        raise ContractError("cache_from_trace: mask length mismatch")
    m = m.to(torch.int32).contiguous()
    ws = _workspace_for(cache, 1)
    cd = cache.desc()
    counts = torch.empty(cache.n_heads, dtype=torch.int32, device=cache.keys.device)
    _check(lib().lkv_mask_counts(C.byref(cd), _ptr(m), m.shape[1], _ptr(counts), C.c_void_p(ws.ptr), ws.nbytes,
                                 _stream()))
    cap = int(counts.sum().item()) + cache.n_heads * decode_slack
    rc = _ragged_for(cache, cap, decode_slack)
    rd = rc.desc()
    _check(lib().lkv_cache_from_trace(C.byref(cd), _ptr(m), m.shape[1], C.byref(rd), C.c_void_p(ws.ptr), ws.nbytes,
                                      _stream()))
    ws.status()
    rc.tokens_seen.copy_(torch.tensor(cache.seq_lens, dtype=torch.int32))
    return rc


# ---- fused eviction ------------------------------------------------------------------------------------
@dataclass
class EvictResult:
    cache: RaggedCache
    scores: torch.Tensor | None
    ratios: torch.Tensor
    budgets: torch.Tensor


class Evictor:
    """Reusable fused eviction (budgets -> score -> select -> compact) with its buffers
    allocated once -- the serving-loop form of prefill_with_eviction's compaction."""

    def __init__(self, cache: DenseCache, scorers: Scorers, logits: torch.Tensor, target_ratio: float,
                 mode: int = BUDGET_EXACT, decode_slack: int = 0, keep_scores: bool = False):
        self.cache, self.scorers = cache, scorers
        self.logits = logits.to(torch.float64).contiguous()
        self.R, self.mode = float(target_ratio), mode
        n_seq, L, H, T, D = cache.shape
        if self.logits.numel() != L * H:
            raise ContractError("one LKV-H logit per (layer, kv head) required")
        cd = cache.desc()
        cap = lib().lkv_ragged_capacity(C.byref(cd), self.R, decode_slack)
        if cap < 0:
            _check(_abi.CONTRACT)
        self.ragged = _ragged_for(cache, cap, decode_slack)
        self.ws = _workspace_for(cache, L * H)
        dev = cache.keys.device
        self.scores = torch.zeros(n_seq, L, H, T, dtype=torch.float32, device=dev) if keep_scores else None
        self.ratios = torch.empty(L * H, dtype=torch.float64, device=dev)
        self.budgets = torch.empty(n_seq, L * H, dtype=torch.int32, device=dev)
        self._cd, self._sd, self._rd = cd, scorers.desc(), self.ragged.desc()

    def launch(self, stream=None) -> None:
        """Enqueue one eviction on `stream` (no host sync; errors latch in the workspace)."""
        _check(lib().lkv_evict(C.byref(self._cd), C.byref(self._sd), _ptr(self.logits), self.R, self.mode,
                               C.byref(self._rd), _ptr(self.scores), _ptr(self.ratios), _ptr(self.budgets),
                               C.c_void_p(self.ws.ptr), self.ws.nbytes, _stream(stream)))

    def launch_host(self, host_keys: torch.Tensor, host_values: torch.Tensor, host_out: "RaggedCache | None" = None,
                    layers_per_chunk: int = 4, stream=None) -> None:
        """Enqueue one eviction of a cache held in pinned host memory (lkv_evict_host): K is
        streamed into this evictor's device K buffer chunk by chunk while earlier chunks are
        scored, kept V rows are gathered straight from host memory, and the compacted cache is
        copied into `host_out` (pinned, same capacity) when given."""
        if not (host_keys.is_pinned() and host_values.is_pinned()):
            raise ContractError("host K/V must be pinned (torch pin_memory)")
        if tuple(host_keys.shape) != self.cache.shape or host_keys.dtype != self.cache.keys.dtype:
            raise ContractError("host K/V must match the evictor's cache shape and dtype")
        hd = CacheDesc(*[getattr(self._cd, f) for f, _ in CacheDesc._fields_])
        hd.keys, hd.values = host_keys.data_ptr(), host_values.data_ptr()
        dev_v = self.cache.values.data_ptr() if self.scorers.input == SCORER_KV else None
        ho = host_out.desc() if host_out is not None else None
        _check(lib().lkv_evict_host(C.byref(hd), C.c_void_p(self.cache.keys.data_ptr()), C.c_void_p(dev_v) if dev_v else None,
                                    C.byref(self._sd), _ptr(self.logits), self.R, self.mode, C.byref(self._rd),
                                    C.byref(ho) if ho is not None else None, layers_per_chunk,
                                    C.c_void_p(self.ws.ptr), self.ws.nbytes, _stream(stream)))

    def host_result_buffer(self) -> "RaggedCache":
        """A pinned host RaggedCache with this evictor's capacity (target of launch_host)."""
        r = self.ragged
        return RaggedCache(r.n_seq, r.n_layers, r.n_kv_heads, r.head_dim, r.dtype, r.capacity_rows, r.decode_slack,
                           device="cpu", pinned=True)

    def run(self) -> EvictResult:
        self.launch()
        self.ws.status()
        self.ragged.tokens_seen.copy_(torch.tensor(self.cache.seq_lens, dtype=torch.int32))
        return EvictResult(self.ragged, self.scores, self.ratios, self.budgets)


def evict(cache: DenseCache, scorers: Scorers, logits: torch.Tensor, target_ratio: float,
          mode: int = BUDGET_EXACT, decode_slack: int = 0, keep_scores: bool = True) -> EvictResult:
    return Evictor(cache, scorers, logits, target_ratio, mode, decode_slack, keep_scores).run()


def prefill_with_eviction(cache: DenseCache, scorers: Scorers, logits: torch.Tensor, target_ratio: float,
                          mode: int = BUDGET_FLOOR, decode_slack: int = 0) -> tuple[RaggedCache, dict]:
    """evictsim.hpp:74 (K/V-given form): score, select and compact every head; report like SimReport."""
    res = evict(cache, scorers, logits, target_ratio, mode, decode_slack, keep_scores=False)
    n_seq, L, H, T, D = cache.shape
    t = cache.seq_lens
    report = {
        "retained_per_head": res.cache.lens.cpu().tolist(),
        "scoring_ops": int(sum(t) * L * H * (scorers.w1.shape[1] * scorers.w1.shape[2] + 3 * scorers.w1.shape[2])),
        "kv_bytes_full": float(sum(t) * L * H * D * 2 * cache.keys.element_size()),
        "kv_bytes_compressed": float(int(res.cache.lens.sum()) * D * 2 * cache.keys.element_size()),
    }
    report["reduction"] = (report["kv_bytes_full"] / report["kv_bytes_compressed"]
                           if report["kv_bytes_compressed"] > 0 else math.inf)
    return res.cache, report


# ---- K5: decode ------------------------------------------------------------------------------------------
def decode_plan(ragged: RaggedCache, group_size: int, rows_per_item: int = 0) -> None:
    """Split every head into attention work items (rows_per_item 0: the plan's choice for one
    all-layer launch; else a multiple of 64 in [128, 1024])."""
    rd = ragged.desc()
    nbytes = lib().lkv_decode_workspace_bytes(C.byref(rd), group_size)
    ragged._decode_ws = Workspace(nbytes, device=ragged.device)
    ragged._decode_G = group_size
    _check(lib().lkv_decode_plan_ex(C.byref(rd), int(rows_per_item), C.c_void_p(ragged._decode_ws.ptr),
                                    ragged._decode_ws.nbytes, _stream()))


def decode_plan_info(ragged: RaggedCache, ws: Workspace | None = None) -> tuple[int, int]:
    """(work items, rows per item) of the current decode plan (or of a model plan's workspace)."""
    ws = ws or ragged._decode_ws
    if ws is None:
        raise ContractError("no decode plan")
    n, ch = C.c_int32(0), C.c_int32(0)
    rd = ragged.desc()
    _check(lib().lkv_decode_plan_info(C.byref(rd), C.c_void_p(ws.ptr), C.byref(n), C.byref(ch), _stream()))
    return int(n.value), int(ch.value)


def decode_step(ragged: RaggedCache, q: torch.Tensor, new_k: torch.Tensor, new_v: torch.Tensor,
                scale: float | None = None, out: torch.Tensor | None = None, check: bool = True) -> torch.Tensor:
    """model.hpp:95's attention block for every (seq, layer): append k/v, attend.
    q: [n_seq, L, Hq, D]; new_k/new_v: [n_seq, L, H, D]."""
    n_seq, L, Hq, D = q.shape
    H = ragged.n_kv_heads
    G = Hq // H
    if ragged._decode_ws is None or ragged._decode_G != G:
        decode_plan(ragged, G)
    if out is None:
        out = torch.empty_like(q)
    scale = scale if scale is not None else 1.0 / math.sqrt(D)
    rd = ragged.desc()
    ws = ragged._decode_ws
    # bind the contiguous copies first: a temporary freed inside the argument list could be handed
    # to the next .contiguous() of the same call before the kernel reads it
    q, new_k, new_v = q.contiguous(), new_k.contiguous(), new_v.contiguous()
    _check(lib().lkv_decode_step(C.byref(rd), n_seq, L, H, Hq, _ptr(q), _ptr(new_k),
                                 _ptr(new_v), _ptr(ragged.tokens_seen), _ptr(out), float(scale),
                                 C.c_void_p(ws.ptr), ws.nbytes, _stream()))
    if check:
        ws.status()
    return out


# ---- evictsim.cpp:56-81 -----------------------------------------------------------------------------------
def kv_memory_bytes(n_layers=32, n_kv_heads=8, head_dim=128, bytes_per_element=2.0, tokens=200000,
                    retention=None, budgets=None) -> dict:
    if n_layers < 1 or n_kv_heads < 1 or head_dim < 1 or tokens < 1 or not bytes_per_element > 0:
        raise ContractError("memory model: all extents must be positive")
    full = float(n_layers) * n_kv_heads * head_dim * 2.0 * bytes_per_element * float(tokens)
    if budgets is not None:
        b = [int(x) for x in budgets]
        if len(b) != n_layers * n_kv_heads:
            raise ContractError("kv_memory_bytes: one budget per head required")
        comp = float(sum(b)) * head_dim * 2.0 * bytes_per_element
        return {"full_bytes": full, "compressed_bytes": comp, "reduction_factor": full / comp if comp else math.inf}
    if not (retention > 0.0) or retention > 1.0:
        raise BudgetError("kv_memory_bytes: retention must lie in (0, 1]")
    comp = retention * full
    return {"full_bytes": full, "compressed_bytes": comp, "reduction_factor": full / comp}
