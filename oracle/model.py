"""fp64 restatement of the reference's toy GQA model decode step -- TEST INFRASTRUCTURE ONLY.

SURVEY 8(f) row 3 (the step after the eviction path): projections, RoPE at ``tokens_seen``,
decode attention over the compacted cache, MLP and logits.  Follows
``proj/src/model.cpp``:

* ``rope_row``      model.cpp:38-46   interleaved pairs, theta = pos * base^(-2j/d)
* ``rmsnorm_row``   model.cpp:48-53   x * gain / sqrt(mean(x^2) + 1e-6)
* ``decode_step``   model.cpp:209-287 append-then-attend per KV head, G = Hq / H,
                                      causal = false, scale 1/sqrt(d); SwiGLU MLP; logits
* ``forward_full``  model.cpp:55-122  full causal forward (used to build prefill caches)

Parameters use the reference's names and layouts (model.cpp:142-163, model.hpp:35-47):
``tok_embed`` [vocab][dm], ``layers.{l}.wq`` [dm][dm], ``wk``/``wv`` [dm][H*d], ``wo``
[dm][dm], ``attn_norm``/``mlp_norm`` [dm], ``w_gate``/``w_up`` [dm][dff], ``w_down``
[dff][dm], ``final_norm`` [dm], ``lm_head`` [dm][vocab].

Pinned against the reference's own model.cpp (compiled into ``oracle/_ref``) by
``tests/test_oracle.py``; ``RefModel`` drives that compiled reference.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np


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
    def d_model(self):
        return self.n_query_heads * self.head_dim

    @property
    def group_size(self):
        return self.n_query_heads // self.n_kv_heads

    @property
    def total_kv_heads(self):
        return self.n_layers * self.n_kv_heads

    @property
    def mlp_width(self):
        return self.mlp_hidden if self.mlp_hidden > 0 else 2 * self.d_model


def param_shapes(cfg: ModelConfig):
    """name -> shape, in the reference's named_params order (model.cpp:142-163)."""
    dm, dkv, dff = cfg.d_model, cfg.n_kv_heads * cfg.head_dim, cfg.mlp_width
    out = {"tok_embed": (cfg.vocab_size, dm)}
    for l in range(cfg.n_layers):
        p = f"layers.{l}."
        out.update({p + "wq": (dm, dm), p + "wk": (dm, dkv), p + "wv": (dm, dkv), p + "wo": (dm, dm),
                    p + "attn_norm": (dm,), p + "mlp_norm": (dm,), p + "w_gate": (dm, dff),
                    p + "w_up": (dm, dff), p + "w_down": (dff, dm)})
    out["final_norm"] = (dm,)
    out["lm_head"] = (dm, cfg.vocab_size)
    return out


def random_params(cfg: ModelConfig, seed: int, gain: float = 0.02, norm_jitter: float = 0.0):
    """Normal(0, gain) matrices, unit norms (+ optional jitter) -- init_model's distribution
    (model.cpp:173-198) from a numpy stream."""
    rng = np.random.default_rng(seed)
    out = {}
    for name, shape in param_shapes(cfg).items():
        if name.endswith("norm"):
            out[name] = 1.0 + norm_jitter * rng.standard_normal(shape)
        else:
            out[name] = gain * rng.standard_normal(shape)
    return out


def rope_row(v: np.ndarray, pos: int, base: float = 10000.0) -> np.ndarray:  # model.cpp:38-46
    d = v.shape[-1]
    j = np.arange(d // 2)
    th = pos * np.power(base, -2.0 * j / d)
    cs, sn = np.cos(th), np.sin(th)
    a, b = v[..., 0::2].copy(), v[..., 1::2].copy()
    out = np.empty_like(v)
    out[..., 0::2] = a * cs - b * sn
    out[..., 1::2] = a * sn + b * cs
    return out


def rmsnorm_row(x: np.ndarray, gain: np.ndarray, eps: float = 1e-6) -> np.ndarray:  # model.cpp:48-53
    ms = np.sum(x * x, axis=-1, keepdims=True)
    return x * gain / np.sqrt(ms / x.shape[-1] + eps)


def _attend(q: np.ndarray, keys: np.ndarray, values: np.ndarray, scale: float) -> np.ndarray:
    """masked_attention_dense with n_q = 1, causal = false, no mask (attention.cpp:46-94)."""
    s = scale * (keys @ q)
    w = np.exp(s - s.max())
    w /= w.sum()
    return w @ values


@dataclass
class HeadCache:  # model.hpp:55-60
    keys: np.ndarray       # [retained][d] fp64, rotary applied
    values: np.ndarray     # [retained][d]
    positions: np.ndarray  # [retained] int


def decode_step(cfg: ModelConfig, P: dict, heads: list, tokens_seen: int, token: int):
    """model.cpp:209-287.  heads: list of HeadCache, layer-major (l * H + h); mutated
    (the new row appended).  Returns (logits [vocab], tokens_seen + 1)."""
    if not (0 <= token < cfg.vocab_size):
        raise ValueError("decode_step: token id out of vocab")
    pos = tokens_seen
    d, H, Hq, G = cfg.head_dim, cfg.n_kv_heads, cfg.n_query_heads, cfg.group_size
    scale = 1.0 / np.sqrt(float(d))
    x = np.array(P["tok_embed"][token], dtype=np.float64)
    for l in range(cfg.n_layers):
        p = f"layers.{l}."
        h = rmsnorm_row(x, P[p + "attn_norm"])
        q = h @ P[p + "wq"]
        k = h @ P[p + "wk"]
        v = h @ P[p + "wv"]
        for kh in range(H):
            hc = heads[l * H + kh]
            kr = rope_row(k[kh * d:(kh + 1) * d], pos)
            hc.keys = np.vstack([hc.keys.reshape(-1, d), kr[None]])
            hc.values = np.vstack([hc.values.reshape(-1, d), v[kh * d:(kh + 1) * d][None]])
            hc.positions = np.append(hc.positions, pos)
        attn = np.empty(cfg.d_model)
        for qh in range(Hq):
            hc = heads[l * H + qh // G]
            qr = rope_row(q[qh * d:(qh + 1) * d], pos)
            attn[qh * d:(qh + 1) * d] = _attend(qr, hc.keys, hc.values, scale)
        x = x + attn @ P[p + "wo"]
        h2 = rmsnorm_row(x, P[p + "mlp_norm"])
        g1 = h2 @ P[p + "w_gate"]
        g2 = h2 @ P[p + "w_up"]
        x = x + (g1 / (1.0 + np.exp(-g1)) * g2) @ P[p + "w_down"]
    logits = rmsnorm_row(x, P["final_norm"]) @ P["lm_head"]
    return logits, pos + 1


def forward_full(cfg: ModelConfig, P: dict, tokens):
    """model.cpp:55-122 without masks: (logits [t][vocab], keys [L*H][t][d], values [L*H][t][d])."""
    tokens = np.asarray(tokens)
    t = len(tokens)
    d, H, Hq, G = cfg.head_dim, cfg.n_kv_heads, cfg.n_query_heads, cfg.group_size
    scale = 1.0 / np.sqrt(float(d))
    pos = np.arange(t)
    x = P["tok_embed"][tokens].astype(np.float64)
    K = np.empty((cfg.total_kv_heads, t, d))
    V = np.empty_like(K)
    causal = np.tril(np.ones((t, t), bool))
    for l in range(cfg.n_layers):
        p = f"layers.{l}."
        h = rmsnorm_row(x, P[p + "attn_norm"])
        q, k, v = h @ P[p + "wq"], h @ P[p + "wk"], h @ P[p + "wv"]
        for kh in range(H):
            K[l * H + kh] = np.stack([rope_row(k[i, kh * d:(kh + 1) * d], i) for i in pos])
            V[l * H + kh] = v[:, kh * d:(kh + 1) * d]
        outs = np.empty((t, cfg.d_model))
        for qh in range(Hq):
            kh = qh // G
            qr = np.stack([rope_row(q[i, qh * d:(qh + 1) * d], i) for i in pos])
            s = scale * qr @ K[l * H + kh].T
            s = np.where(causal, s, -np.inf)
            w = np.exp(s - s.max(axis=1, keepdims=True))
            w /= w.sum(axis=1, keepdims=True)
            outs[:, qh * d:(qh + 1) * d] = w @ V[l * H + kh]
        x = x + outs @ P[p + "wo"]
        h2 = rmsnorm_row(x, P[p + "mlp_norm"])
        g1, g2 = h2 @ P[p + "w_gate"], h2 @ P[p + "w_up"]
        x = x + (g1 / (1.0 + np.exp(-g1)) * g2) @ P[p + "w_down"]
    logits = rmsnorm_row(x, P["final_norm"]) @ P["lm_head"]
    return logits, K, V


class RefModel:
    """The reference's own ModelWeights / forward_full / decode_step (oracle/_ref)."""

    def __init__(self, cfg: ModelConfig):
        from . import ref_lib

        R = ref_lib()
        if R is None:
            raise RuntimeError("oracle/_ref not built")
        R.ref_model_create.restype = C.c_void_p
        R.ref_model_create.argtypes = [C.c_int] * 7 + [C.c_ulonglong]
        R.ref_model_free.argtypes = [C.c_void_p]
        R.ref_model_param_numel.restype = C.c_long
        R.ref_model_param_numel.argtypes = [C.c_void_p, C.c_char_p]
        R.ref_model_get.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p, C.c_long]
        R.ref_model_set.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p, C.c_long]
        R.ref_forward_full.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        R.ref_decode_steps.argtypes = [C.c_void_p] + [C.c_void_p] * 5 + [C.c_int, C.c_void_p, C.c_int] + \
            [C.c_void_p] * 4
        self.R, self.cfg = R, cfg
        self.h = R.ref_model_create(cfg.n_layers, cfg.n_query_heads, cfg.n_kv_heads, cfg.head_dim, cfg.vocab_size,
                                    cfg.max_seq_len, cfg.mlp_hidden, cfg.rng_seed)
        if not self.h:
            raise RuntimeError("ref_model_create failed")

    def __del__(self):
        if getattr(self, "h", None):
            self.R.ref_model_free(self.h)
            self.h = None

    def params(self) -> dict:
        out = {}
        for name, shape in param_shapes(self.cfg).items():
            a = np.empty(shape, np.float64)
            assert self.R.ref_model_get(self.h, name.encode(), a.ctypes.data, a.size) == 0
            out[name] = a
        return out

    def set_params(self, P: dict) -> None:
        for name in param_shapes(self.cfg):
            a = np.ascontiguousarray(P[name], np.float64)
            assert self.R.ref_model_set(self.h, name.encode(), a.ctypes.data, a.size) == 0, name

    def forward_full(self, tokens):
        c = self.cfg
        tok = np.ascontiguousarray(tokens, np.int32)
        t = len(tok)
        logits = np.empty((t, c.vocab_size))
        K = np.empty((c.total_kv_heads, t, c.head_dim))
        V = np.empty_like(K)
        rc = self.R.ref_forward_full(self.h, tok.ctypes.data, t, logits.ctypes.data, K.ctypes.data, V.ctypes.data)
        if rc:
            raise RuntimeError(f"ref_forward_full: status {rc}")
        return logits, K, V

    def decode_steps(self, heads: list, tokens_seen: int, tokens):
        """Runs decode_step len(tokens) times on a cache built from `heads` (HeadCache list).
        Returns (logits [n][vocab], new_k [n][L*H][d], new_v, tokens_seen)."""
        c = self.cfg
        d, n = c.head_dim, c.total_kv_heads
        lens = np.array([len(h.positions) for h in heads], np.int32)
        off = np.zeros(n, np.int64)
        off[1:] = np.cumsum(lens)[:-1]
        rows = max(int(lens.sum()), 1)
        K = np.zeros((rows, d))
        V = np.zeros((rows, d))
        pos = np.zeros(rows, np.int32)
        for i, h in enumerate(heads):
            K[off[i]:off[i] + lens[i]] = h.keys.reshape(-1, d)
            V[off[i]:off[i] + lens[i]] = h.values.reshape(-1, d)
            pos[off[i]:off[i] + lens[i]] = h.positions
        tok = np.ascontiguousarray(tokens, np.int32)
        ns = len(tok)
        logits = np.empty((ns, c.vocab_size))
        nk = np.empty((ns, n, d))
        nv = np.empty((ns, n, d))
        ts = C.c_int32(0)
        rc = self.R.ref_decode_steps(self.h, lens.ctypes.data, off.ctypes.data, K.ctypes.data, V.ctypes.data,
                                     pos.ctypes.data, tokens_seen, tok.ctypes.data, ns, logits.ctypes.data,
                                     nk.ctypes.data, nv.ctypes.data, C.addressof(ts))
        if rc:
            raise RuntimeError(f"ref_decode_steps: status {rc}")
        return logits, nk, nv, ts.value
