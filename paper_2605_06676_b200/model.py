"""Full decode step of the reference's toy GQA model on the B200.

Host mirror of ``ModelConfig`` / ``ModelWeights`` / ``decode_step`` (``model.hpp:18-47,95``,
``model.cpp:209-287``) over the C ABI ``lkv_model_*`` (``include/lkv_b200.h``).  The step after
the eviction path: after ``lkv_evict`` compacts the prefill cache, every decode step runs the
projections (weight-streaming tensor-core GEMVs with fused RoPE / residual / SwiGLU epilogues),
the per-layer decode attention over the compacted ragged cache (K5), and the logits -- all on the
device, one stream, PDL-chained launches that capture into a CUDA graph.

Parameters are given by the reference's names and layouts (``model.cpp:142-163``):
``tok_embed``, ``layers.{l}.wq|wk|wv|wo|attn_norm|mlp_norm|w_gate|w_up|w_down``, ``final_norm``,
``lm_head``, each ``x W`` row-major.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import RaggedCache, Workspace, _check, _dtype_code, _ptr, _stream, lib
from ._abi import (MODEL_MAX_SEQ, P_ATTN_NORM, P_FINAL_NORM, P_LM_HEAD, P_MLP_NORM, P_TOK_EMBED, P_W_DOWN, P_W_GATE,
                   P_W_UP, P_WK, P_WO, P_WQ, P_WV, ModelDesc)


@dataclass
class ModelConfig:  # model.hpp:18-32
    n_layers: int = 4
    n_query_heads: int = 8
    n_kv_heads: int = 2
    head_dim: int = 16
    vocab_size: int = 256
    max_seq_len: int = 512
    rng_seed: int = 1234
    mlp_hidden: int = 0

    @property
    def d_model(self) -> int:
        return self.n_query_heads * self.head_dim

    @property
    def group_size(self) -> int:
        return self.n_query_heads // self.n_kv_heads

    @property
    def total_kv_heads(self) -> int:
        return self.n_layers * self.n_kv_heads

    @property
    def mlp_width(self) -> int:
        return self.mlp_hidden if self.mlp_hidden > 0 else 2 * self.d_model


_LAYER_PARAMS = {"wq": P_WQ, "wk": P_WK, "wv": P_WV, "wo": P_WO, "attn_norm": P_ATTN_NORM, "mlp_norm": P_MLP_NORM,
                 "w_gate": P_W_GATE, "w_up": P_W_UP, "w_down": P_W_DOWN}
_GLOBAL_PARAMS = {"tok_embed": P_TOK_EMBED, "final_norm": P_FINAL_NORM, "lm_head": P_LM_HEAD}


def param_names(cfg: ModelConfig):
    """The reference's named_params order (model.cpp:142-163)."""
    out = ["tok_embed"]
    for l in range(cfg.n_layers):
        out += [f"layers.{l}.{n}" for n in ("wq", "wk", "wv", "wo", "attn_norm", "mlp_norm", "w_gate", "w_up",
                                            "w_down")]
    return out + ["final_norm", "lm_head"]


def _param_kind(name: str):
    if name in _GLOBAL_PARAMS:
        return _GLOBAL_PARAMS[name], 0
    parts = name.split(".")
    if len(parts) != 3 or parts[0] != "layers" or parts[2] not in _LAYER_PARAMS:
        raise KeyError(f"unknown model parameter {name!r}")
    return _LAYER_PARAMS[parts[2]], int(parts[1])


class DecodeModel:
    """ModelWeights resident in HBM in the library's packed layout + decode_step."""

    def __init__(self, cfg: ModelConfig, params: dict, dtype=torch.bfloat16, device="cuda",
                 rope_base: float = 10000.0, norm_eps: float = 1e-6):
        self.cfg, self.dtype, self.device = cfg, dtype, device
        self.desc = ModelDesc(cfg.n_layers, cfg.n_query_heads, cfg.n_kv_heads, cfg.head_dim, cfg.vocab_size,
                              cfg.max_seq_len, cfg.mlp_width, _dtype_code(dtype), float(rope_base), float(norm_eps))
        _check(lib().lkv_model_validate(C.byref(self.desc)))
        nbytes = lib().lkv_model_weights_bytes(C.byref(self.desc))
        self.weights = torch.zeros(nbytes, dtype=torch.uint8, device=device)
        missing = set(param_names(cfg)) - set(params)
        if missing:
            raise KeyError(f"missing model parameters: {sorted(missing)[:4]}...")
        s = _stream()
        for name, t in params.items():
            kind, layer = _param_kind(name)
            src = torch.as_tensor(t).to(device=device, dtype=dtype).contiguous()
            _check(lib().lkv_model_load_param(C.byref(self.desc), _ptr(self.weights), kind, layer, _ptr(src), s))
        torch.cuda.current_stream().synchronize()
        self.cache = None
        self.ws = None

    def bind(self, cache: RaggedCache, rows_per_item: int = 0) -> None:
        """Attach a compacted cache (after every eviction): plans the per-layer attention
        work (rows_per_item 0: one wave per layer; else fixed) and builds the RoPE table."""
        if cache.n_seq > MODEL_MAX_SEQ:
            raise ValueError(f"at most {MODEL_MAX_SEQ} sequences per decode batch")
        rd = cache.desc()
        nbytes = lib().lkv_model_workspace_bytes(C.byref(self.desc), cache.n_seq, C.byref(rd))
        if nbytes == 0:
            _check(1)
        self.cache = cache
        self.ws = Workspace(nbytes, device=self.device)
        _check(lib().lkv_model_plan_ex(C.byref(self.desc), C.byref(rd), cache.n_seq, int(rows_per_item),
                                       C.c_void_p(self.ws.ptr), self.ws.nbytes, _stream()))
        self._rd = rd

    def step(self, tokens: torch.Tensor, logits: torch.Tensor | None = None, check: bool = True) -> torch.Tensor:
        """decode_step (model.cpp:209-287) for every bound sequence: tokens [n_seq] int32 (device).
        Appends one row to every head of the cache, advances tokens_seen, returns fp32 logits
        [n_seq][vocab]."""
        c = self.cache
        if c is None:
            raise RuntimeError("bind() a cache first")
        if logits is None:
            logits = torch.empty(c.n_seq, self.cfg.vocab_size, dtype=torch.float32, device=self.device)
        _check(lib().lkv_model_decode_step(C.byref(self.desc), _ptr(self.weights), C.byref(self._rd), c.n_seq,
                                           _ptr(tokens), _ptr(c.tokens_seen), _ptr(logits),
                                           C.c_void_p(self.ws.ptr), self.ws.nbytes, _stream()))
        if check:
            self.ws.status()
        return logits

    def capture(self, tokens: torch.Tensor, logits: torch.Tensor) -> torch.cuda.CUDAGraph:
        """One decode step captured as a CUDA graph reading `tokens` and writing `logits`
        (static buffers); replay() runs a step with ~no launch overhead.  The cache state is
        unchanged by the capture (the warm-up step's append is rolled back)."""
        c = self.cache
        lens, seen = c.lens.clone(), c.tokens_seen.clone()
        self.step(tokens, logits, check=False)  # warm (attributes, lazy init) outside capture
        c.lens.copy_(lens)
        c.tokens_seen.copy_(seen)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.step(tokens, logits, check=False)
        return g
