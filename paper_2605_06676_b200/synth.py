"""Seeded synthetic inputs for the BASELINE.json configs (harness, not product).

The reference measures on LongBench/RULER-style prompts through a Llama model;
none of that is in this container, so seeded synthetic tensors with the
configs' shapes and value distributions stand in (BASELINE.json `configs`,
SURVEY.md 8(d)):

  K, V ~ N(0, 1) with 4 outlier channels x8 (per (layer, head) for C1, per layer
  otherwise, the same channels for K and V); scorer 128 -> 64 -> 1 GELU with
  W1, w2 ~ N(0, 0.02), b1 = 0 (one scorer per layer); LKV-H logits ~ N(0, sigma);
  q, new k/v ~ N(0, 1).  Keys are treated as already post-RoPE.

Everything is generated on the device from a torch Generator seeded with
1000 + config id; the oracle sees the very same buffers (downloaded).
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from . import GELU_ERF, SCORER_K, DenseCache, Scorers


@dataclass(frozen=True)
class Config:
    cid: int
    n_layers: int
    n_kv_heads: int
    n_q_heads: int
    head_dim: int
    max_tokens: int
    n_seq: int
    dtype: torch.dtype
    ratio: float
    logit_sigma: float = 1.0
    hidden: int = 64
    decode_steps: int = 128
    ragged_lo: int = 0  # >0: per-sequence lengths ~ U[ragged_lo, max_tokens]
    per_head_outliers: bool = False

    @property
    def name(self):
        return f"C{self.cid}"


CONFIGS = {
    1: Config(1, 1, 8, 32, 128, 4096, 1, torch.float32, 0.15, decode_steps=1, per_head_outliers=True),
    2: Config(2, 32, 8, 32, 128, 32768, 1, torch.bfloat16, 0.15, decode_steps=128),
    3: Config(3, 32, 8, 32, 128, 131072, 1, torch.bfloat16, 0.15, decode_steps=128),
    4: Config(4, 32, 8, 32, 128, 32768, 16, torch.bfloat16, 0.15, decode_steps=256, ragged_lo=8192),
    5: Config(5, 80, 8, 64, 128, 65536, 4, torch.bfloat16, 0.10, logit_sigma=1.5, decode_steps=128),
}


def seq_lens_for(cfg: Config, seed: int | None = None) -> list:
    if cfg.ragged_lo <= 0:
        return [cfg.max_tokens] * cfg.n_seq
    g = torch.Generator().manual_seed((seed if seed is not None else 1000 + cfg.cid) + 7)
    return torch.randint(cfg.ragged_lo, cfg.max_tokens + 1, (cfg.n_seq,), generator=g).tolist()


def make_cache(cfg: Config, device="cuda", seed: int | None = None, n_layers: int | None = None,
               max_tokens: int | None = None, n_seq: int | None = None) -> DenseCache:
    """K/V [n_seq, L, H, T, D] with outlier channels.  Optional overrides shrink the
    config for parity tests (same distributions)."""
    L = n_layers or cfg.n_layers
    T = max_tokens or cfg.max_tokens
    S = n_seq or cfg.n_seq
    H, D = cfg.n_kv_heads, cfg.head_dim
    seed = 1000 + cfg.cid if seed is None else seed
    g = torch.Generator(device=device).manual_seed(seed)
    gc = torch.Generator().manual_seed(seed + 1)
    K = torch.empty(S, L, H, T, D, dtype=cfg.dtype, device=device)
    V = torch.empty_like(K)
    for l in range(L):
        if cfg.per_head_outliers:
            chans = [torch.randperm(D, generator=gc)[:4] for _ in range(H)]
        else:
            c = torch.randperm(D, generator=gc)[:4]
            chans = [c] * H
        scale = torch.ones(H, 1, D, device=device)
        for h in range(H):
            scale[h, 0, chans[h].to(device)] = 8.0
        for s in range(S):
            for X in (K, V):
                x = torch.randn(H, T, D, generator=g, device=device, dtype=torch.float32)
                X[s, l].copy_((x * scale).to(cfg.dtype))
    lens = seq_lens_for(cfg, seed) if n_seq is None and max_tokens is None else [T] * S
    if cfg.ragged_lo > 0 and (n_seq is not None or max_tokens is not None):
        gl = torch.Generator().manual_seed(seed + 7)
        lo = min(cfg.ragged_lo, T)
        lens = torch.randint(lo, T + 1, (S,), generator=gl).tolist()
    return DenseCache(K, V, lens)


def make_scorers(cfg: Config, device="cuda", seed: int | None = None, n_layers: int | None = None) -> Scorers:
    """One 128 -> hidden -> 1 GELU scorer per layer, W ~ N(0, 0.02), b1 = 0."""
    L = n_layers or cfg.n_layers
    seed = 2000 + cfg.cid if seed is None else seed
    g = torch.Generator(device=device).manual_seed(seed)
    w1 = (torch.randn(L, cfg.head_dim, cfg.hidden, generator=g, device=device) * 0.02).to(cfg.dtype)
    w2 = torch.randn(L, cfg.hidden, generator=g, device=device) * 0.02
    b1 = torch.zeros(L, cfg.hidden, device=device)
    return Scorers(w1, b1, w2, input=SCORER_K, activation=GELU_ERF, stride_layer=1, stride_head=0)


def make_logits(cfg: Config, device="cuda", seed: int | None = None, n_layers: int | None = None) -> torch.Tensor:
    L = n_layers or cfg.n_layers
    seed = 3000 + cfg.cid if seed is None else seed
    g = torch.Generator().manual_seed(seed)
    return (torch.randn(L * cfg.n_kv_heads, generator=g, dtype=torch.float64) * cfg.logit_sigma).to(device)


def make_decode_inputs(cfg: Config, step: int, device="cuda", n_layers: int | None = None,
                       n_seq: int | None = None, seed: int | None = None):
    L = n_layers or cfg.n_layers
    S = n_seq or cfg.n_seq
    seed = (4000 + cfg.cid if seed is None else seed) * 100003 + step
    g = torch.Generator(device=device).manual_seed(seed)
    q = torch.randn(S, L, cfg.n_q_heads, cfg.head_dim, generator=g, device=device).to(cfg.dtype)
    k = torch.randn(S, L, cfg.n_kv_heads, cfg.head_dim, generator=g, device=device).to(cfg.dtype)
    v = torch.randn(S, L, cfg.n_kv_heads, cfg.head_dim, generator=g, device=device).to(cfg.dtype)
    return q, k, v
