"""Layer-by-layer prefill with eviction (evictsim.cpp:131-159).

The reference computes one layer's K/V over the full prefix, scores and compacts that layer
per KV head, then moves on, so the peak KV footprint is ONE full-length layer plus the
compressed earlier layers (the peak accounting of evictsim.cpp:157-159).  Here, per layer:

  lkv_kv_project                    (h [Wk | Wv] on tcgen05 with RoPE at absolute positions and
                                     the token-major -> head-major pack fused in the epilogue,
                                     into ONE reusable dense layer buffer; ingest_layer_hidden)
  or, for projections computed elsewhere, lkv_rope_pack (ingest_layer)
  lkv_score + lkv_select(gather)    (per sequence, with that layer's slice of the budgets that
                                     lkv_budgets solved once over ALL L*H logits)

into one ragged cache whose offsets are global, so the result is the same cache a one-shot
`lkv_evict` over all layers produces (tests/test_gpu_parity.py checks bit-equality).
"""
from __future__ import annotations

import ctypes as C

import torch

from . import (BUDGET_EXACT, CacheDesc, ContractError, DenseCache, RaggedCache, RaggedDesc, ScorerDesc, Scorers,
               Workspace, _check, _ptr, _stream, lib)


class LayerwisePrefill:
    def __init__(self, n_seq: int, n_layers: int, n_kv_heads: int, head_dim: int, max_tokens: int, seq_lens,
                 scorers: Scorers, logits: torch.Tensor, target_ratio: float, mode: int = BUDGET_EXACT,
                 decode_slack: int = 0, dtype=torch.bfloat16, rope_base: float = 10000.0, device="cuda"):
        self.S, self.L, self.H, self.D, self.T = n_seq, n_layers, n_kv_heads, head_dim, max_tokens
        self.seq_lens = [int(t) for t in seq_lens]
        self.dtype, self.device, self.scorers = dtype, device, scorers
        self.logits = logits.to(torch.float64).contiguous()
        if self.logits.numel() != n_layers * n_kv_heads:
            raise ContractError("one LKV-H logit per (layer, kv head) required")
        self.R, self.mode = float(target_ratio), mode
        # one reusable dense layer (the only full-length KV ever resident)
        self.k_layer = torch.empty(n_seq, 1, n_kv_heads, max_tokens, head_dim, dtype=dtype, device=device)
        self.v_layer = torch.empty_like(self.k_layer)
        self.layer = DenseCache(self.k_layer, self.v_layer, self.seq_lens)
        full_desc = CacheDesc(n_seq, n_layers, n_kv_heads, head_dim, max_tokens, self.layer.desc().dtype, 0, None, None,
                              self.layer.desc().seq_lens)
        cap = lib().lkv_ragged_capacity(C.byref(full_desc), self.R, decode_slack)
        if cap < 0:
            _check(1)
        self.ragged = RaggedCache(n_seq, n_layers, n_kv_heads, head_dim, dtype, cap, decode_slack, device=device)
        self.budgets = torch.empty(n_seq, n_layers * n_kv_heads, dtype=torch.int32, device=device)
        self.ratios = torch.empty(n_layers * n_kv_heads, dtype=torch.float64, device=device)
        self.table = torch.empty(max_tokens, head_dim // 2, 2, dtype=torch.float32, device=device)
        # per-(sequence, layer) views share one workspace sized for a single sequence-layer
        one = DenseCache(self.k_layer[:1], self.v_layer[:1], self.seq_lens[:1])
        self._ws = Workspace(lib().lkv_workspace_bytes(C.byref(one.desc()), 1), device=device)
        self._bws = Workspace(256, device=device)
        self.scores = torch.empty(1, 1, n_kv_heads, max_tokens, dtype=torch.float32, device=device)
        self.dense_layer_bytes = 2 * self.k_layer.numel() * self.k_layer.element_size()
        self.peak_kv_bytes = 0
        self._ingested = 0
        self._budget_prefix = None
        s = _stream()
        lens_c = (C.c_int32 * n_seq)(*self.seq_lens)
        _check(lib().lkv_rope_table(max_tokens, head_dim, float(rope_base), 0, _ptr(self.table), s))
        _check(lib().lkv_budgets(_ptr(self.logits), n_layers * n_kv_heads, self.R, mode, lens_c, n_seq, decode_slack,
                                 _ptr(self.ratios), _ptr(self.budgets), _ptr(self.ragged.offsets),
                                 C.c_void_p(self._bws.ptr), self._bws.nbytes, s))

    def ingest_layer_hidden(self, l: int, h: torch.Tensor, wkv_t: torch.Tensor) -> None:
        """Produce layer `l`'s K/V from the attention-normed hidden states h [n_seq, max_tokens,
        d_model] and the transposed [Wk | Wv] weights wkv_t [2 * H * D, d_model] (kv_weights())
        with lkv_kv_project (tcgen05 GEMM, RoPE + head-major pack fused), then score, select and
        compact it."""
        S, H, D, T = self.S, self.H, self.D, self.T
        if h.dim() != 3 or h.shape[:2] != (S, T) or h.dtype != self.dtype or wkv_t.shape != (2 * H * D, h.shape[2]):
            raise ContractError("h must be [n_seq, max_tokens, d_model] and wkv_t [2 * H * D, d_model]")
        ld = self.layer.desc()
        h, wkv_t = h.contiguous(), wkv_t.contiguous()  # alive across the call
        _check(lib().lkv_kv_project(_ptr(h), h.shape[2], _ptr(wkv_t), C.byref(ld),
                                    _ptr(self.table), _ptr(self.k_layer), _ptr(self.v_layer), _stream()))
        self._score_select(l)

    def ingest_layer(self, l: int, k_lin: torch.Tensor, v_lin: torch.Tensor) -> None:
        """Rope, score, select and compact layer `l` from its projections
        k_lin / v_lin [n_seq, max_tokens, n_kv_heads * head_dim] (post-GEMM, pre-RoPE)."""
        S, H, D, T = self.S, self.H, self.D, self.T
        if k_lin.shape != (S, T, H * D) or v_lin.shape != k_lin.shape or k_lin.dtype != self.dtype:
            raise ContractError("projections must be [n_seq, max_tokens, n_kv_heads * head_dim] in the cache dtype")
        k_lin, v_lin = k_lin.contiguous(), v_lin.contiguous()
        s = _stream()
        ld = self.layer.desc()
        _check(lib().lkv_rope_pack(_ptr(k_lin), _ptr(v_lin), C.byref(ld), _ptr(self.table), _ptr(self.k_layer),
                                   _ptr(self.v_layer), s))
        self._score_select(l)

    def _score_select(self, l: int) -> None:
        S, H, D, T = self.S, self.H, self.D, self.T
        s = _stream()
        ld = self.layer.desc()
        sc = self.scorers
        in_dim = sc.w1.shape[1]
        hidden = sc.w1.shape[2]
        esz = sc.w1t.element_size()
        sc0 = l * sc.stride_layer
        sd = ScorerDesc(sc.input, sc.activation, hidden, sc.w1.shape[0] - sc0, sc.stride_layer, sc.stride_head,
                        sc.w1t.data_ptr() + sc0 * hidden * in_dim * esz, sc.b1.data_ptr() + sc0 * hidden * 4,
                        sc.w2.data_ptr() + sc0 * hidden * 4)
        r = self.ragged
        for q in range(S):
            lens_q = (C.c_int32 * 1)(self.seq_lens[q])
            cd = CacheDesc(1, 1, H, D, T, ld.dtype, 0, self.k_layer[q].data_ptr(), self.v_layer[q].data_ptr(), lens_q)
            h0 = (q * self.L + l) * H  # first flat head of (q, l) in the global ragged cache
            rd = RaggedDesc(H, D, ld.dtype, r.decode_slack, r.capacity_rows, r.offsets.data_ptr() + 8 * h0,
                            r.lens.data_ptr() + 4 * h0, r.keys.data_ptr(), r.values.data_ptr(), r.positions.data_ptr())
            b = self.budgets[q, l * H:(l + 1) * H]
            # score (top-k histogram fused into the scorer epilogue) -> select -> gather, one call
            _check(lib().lkv_evict_budgets(C.byref(cd), C.byref(sd), _ptr(b), C.byref(rd), _ptr(self.scores),
                                           C.c_void_p(self._ws.ptr), self._ws.nbytes, s))
        self._ingested += 1
        if self._budget_prefix is None:  # one host read of the budgets, for the peak accounting only
            per_layer = self.budgets.reshape(S, self.L, H).sum(dim=(0, 2)).cpu().tolist()
            self._budget_prefix = [sum(per_layer[:i]) for i in range(self.L + 1)]
        compressed = self._budget_prefix[l] * 2 * D * self.k_layer.element_size()
        self.peak_kv_bytes = max(self.peak_kv_bytes, compressed + self.dense_layer_bytes)

    def finish(self) -> RaggedCache:
        if self._ingested != self.L:
            raise ContractError("every layer must be ingested before finish()")
        self._bws.status()
        self._ws.status()
        self.ragged.tokens_seen.copy_(torch.tensor(self.seq_lens, dtype=torch.int32))
        return self.ragged


def rope_table(max_tokens: int, head_dim: int, base: float = 10000.0, pos_offset: int = 0, device="cuda"):
    """cos/sin table [max_tokens, head_dim/2, 2] (fp64-evaluated, stored fp32)."""
    t = torch.empty(max_tokens, head_dim // 2, 2, dtype=torch.float32, device=device)
    _check(lib().lkv_rope_table(max_tokens, head_dim, float(base), pos_offset, _ptr(t), _stream()))
    return t


def kv_weights(wk: torch.Tensor, wv: torch.Tensor) -> torch.Tensor:
    """[Wk | Wv] (reference layout x W, [d_model, H * D] each) -> the transposed, concatenated
    [2 * H * D, d_model] operand lkv_kv_project reads (K-major for the UMMA B operand)."""
    return torch.cat([wk, wv], dim=1).t().contiguous()


def kv_project(h: torch.Tensor, wkv_t: torch.Tensor, table: torch.Tensor, seq_lens, n_kv_heads: int,
               head_dim: int = 128):
    """h [n_seq, T, d_model] bf16 -> (K roped, V) dense layer [n_seq, 1, H, T, D] (lkv_kv_project)."""
    S, T, dm = h.shape
    k_out = torch.empty(S, 1, n_kv_heads, T, head_dim, dtype=h.dtype, device=h.device)
    v_out = torch.empty_like(k_out)
    layer = DenseCache(k_out, v_out, list(seq_lens))
    h, wkv_t = h.contiguous(), wkv_t.contiguous()  # alive across the call
    _check(lib().lkv_kv_project(_ptr(h), dm, _ptr(wkv_t), C.byref(layer.desc()), _ptr(table),
                                _ptr(k_out), _ptr(v_out), _stream()))
    return k_out, v_out


def rope_pack(k_lin: torch.Tensor, v_lin: torch.Tensor, table: torch.Tensor, seq_lens, n_kv_heads: int):
    """[n_seq, T, H*D] projections -> (K roped, V) dense layer [n_seq, 1, H, T, D]."""
    S, T, HD = k_lin.shape
    D = HD // n_kv_heads
    k_out = torch.empty(S, 1, n_kv_heads, T, D, dtype=k_lin.dtype, device=k_lin.device)
    v_out = torch.empty_like(k_out)
    layer = DenseCache(k_out, v_out, list(seq_lens))
    # both contiguous copies alive across the call: two temporaries freed inside one argument list
    # can share a caching-allocator block (the second copy overwrote the first, K came out as V)
    k_lin, v_lin = k_lin.contiguous(), v_lin.contiguous()
    _check(lib().lkv_rope_pack(_ptr(k_lin), _ptr(v_lin), C.byref(layer.desc()), _ptr(table),
                               _ptr(k_out), _ptr(v_out), _stream()))
    return k_out, v_out
