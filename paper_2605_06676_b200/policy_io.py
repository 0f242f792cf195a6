"""Trained-policy ingestion: read the reference's LKV policy
checkpoint (`lkv train` writes `lkv_params.bin`) and turn it into the device path's inputs.

Format (container.cpp:45-76, 92-137; checkpoint.cpp:56-86): an 8-byte little-endian
metadata length, an ordered JSON object {name: {dtype, shape, byte_offset, byte_length}},
then the payloads back to back (f64, or f32 widened to f64 on load).  The policy file holds
`__meta` = [version 1, n_layers, n_kv_heads, d_e, d_head], `head_embeddings` [L*H, d_e],
`head_predictor.{w1,b1,w2}` (d_e -> d_e/2 -> 1) and `token_scorers.<i>.{w1,b1,w2}`
(2 d_head -> d_head -> 1, one per (layer, kv head), policy.hpp:34-47).

`head_scores` (policy.cpp:106-108) runs the head predictor on the device in fp64
(lkv_f64_token_scores: silu(E W1 + b1) w2, mlp2_forward policy.cpp:30-34), so the LKV-H logits
handed to K2 are the reference's own to the last few ulps.
"""
from __future__ import annotations

import json
import struct
from dataclasses import dataclass

import numpy as np

from . import SCORER_KV, SILU, ContractError, Scorers

_VERSION = 1.0


@dataclass
class Mlp2:
    w1: np.ndarray  # [in, hidden]
    b1: np.ndarray  # [hidden]
    w2: np.ndarray  # [hidden]


@dataclass
class LkvParams:
    n_layers: int
    n_kv_heads: int
    d_e: int
    d_head: int
    head_embeddings: np.ndarray
    head_predictor: Mlp2
    token_scorers: list


def load_container(path: str) -> dict:
    """container.cpp:92-137 -- ordered {name: float64 ndarray}; same validation errors."""
    with open(path, "rb") as f:
        raw = f.read()
    if len(raw) < 8:
        raise ContractError("container: truncated header")
    (meta_len,) = struct.unpack("<Q", raw[:8])
    if 8 + meta_len > len(raw):
        raise ContractError("container: truncated metadata")
    try:
        meta = json.loads(raw[8:8 + meta_len].decode("utf-8"))
    except Exception as e:  # noqa: BLE001
        raise ContractError("container: bad metadata JSON") from e
    if not isinstance(meta, dict):
        raise ContractError("container: bad metadata JSON")
    payload = raw[8 + meta_len:]
    out, expected = {}, 0
    for name, m in meta.items():
        if not all(k in m for k in ("dtype", "shape", "byte_offset", "byte_length")):
            raise ContractError("container: incomplete record for " + name)
        dt = {"f64": np.float64, "f32": np.float32}.get(m["dtype"])
        if dt is None:
            raise ContractError("container: unknown dtype " + str(m["dtype"]))
        off, ln, shape = int(m["byte_offset"]), int(m["byte_length"]), [int(x) for x in m["shape"]]
        if off != expected:
            raise ContractError("container: offsets must be contiguous and in order")
        if off + ln > len(payload):
            raise ContractError("container: payload shorter than metadata claims")
        numel = int(np.prod(shape)) if shape else 1
        if ln != numel * np.dtype(dt).itemsize:
            raise ContractError("container: byte length mismatch for " + name)
        out[name] = np.frombuffer(payload, dtype=dt, count=numel, offset=off).astype(np.float64).reshape(shape)
        expected = off + ln
    if expected != len(payload):
        raise ContractError("container: trailing bytes after last tensor")
    return out


def _mlp(c: dict, prefix: str) -> Mlp2:
    return Mlp2(c[prefix + "w1"], c[prefix + "b1"].reshape(-1), c[prefix + "w2"].reshape(-1))


def load_lkv_params(path: str) -> LkvParams:
    """checkpoint.cpp:68-86."""
    c = load_container(path)
    meta = c.get("__meta")
    if meta is None or meta.size != 5 or meta.reshape(-1)[0] != _VERSION:
        raise ContractError("policy checkpoint: unsupported metadata")
    _, L, H, d_e, d = (int(x) for x in meta.reshape(-1))
    n = L * H
    p = LkvParams(L, H, d_e, d, c["head_embeddings"], _mlp(c, "head_predictor."),
                  [_mlp(c, f"token_scorers.{i}.") for i in range(n)])
    if p.head_embeddings.shape != (n, d_e):
        raise ContractError("policy checkpoint: shape mismatch for head_embeddings")
    for i, m in enumerate(p.token_scorers):
        if m.w1.shape != (2 * d, d) or m.b1.shape != (d,) or m.w2.shape != (d,):
            raise ContractError(f"policy checkpoint: shape mismatch for token_scorers.{i}")
    return p


def head_scores(p: LkvParams, device="cuda"):
    """policy.cpp:106-108: silu(E W1 + b1) w2 (mlp2_forward, policy.cpp:30-34), fp64 on the
    device (lkv_f64_token_scores).  Returns a device fp64 tensor [L*H]."""
    import ctypes as C

    import torch

    from . import SCORER_K, Workspace, _check, _ptr, _stream, lib

    def dev(a):
        return torch.tensor(np.ascontiguousarray(a, dtype=np.float64), device=device)

    E, W1, B1, W2 = (dev(x) for x in (p.head_embeddings, p.head_predictor.w1, p.head_predictor.b1,
                                      p.head_predictor.w2))
    n, de = E.shape
    hidden = W1.shape[1]
    u = torch.empty(n, dtype=torch.float64, device=device)
    ws = Workspace(256, device=device)
    _check(lib().lkv_f64_token_scores(n, de, SCORER_K, _ptr(E), de, None, 0, _ptr(W1), _ptr(B1), _ptr(W2), hidden,
                                      SILU, _ptr(u), C.c_void_p(ws.ptr), ws.nbytes, _stream()))
    ws.status()
    return u


def scorers_from_params(p: LkvParams, dtype=None, device="cuda") -> Scorers:
    """The per-(layer, head) token scorers as the device's reference-mode scorer table
    ([k;v] -> d -> 1, SiLU; scorer id = l * H + h, policy.cpp:100-102)."""
    import torch

    dtype = dtype or torch.bfloat16
    w1 = torch.tensor(np.stack([m.w1 for m in p.token_scorers]), dtype=dtype, device=device)
    b1 = torch.tensor(np.stack([m.b1 for m in p.token_scorers]), dtype=torch.float32, device=device)
    w2 = torch.tensor(np.stack([m.w2 for m in p.token_scorers]), dtype=torch.float32, device=device)
    return Scorers(w1, b1, w2, input=SCORER_KV, activation=SILU, stride_layer=p.n_kv_heads, stride_head=1)


# ---- export-budgets (tools/lkv.cpp:154-177, policy.cpp:301-311) ----------------------------------
def budget_table_csv(ratios, n_layers: int, n_kv_heads: int) -> str:
    """policy.cpp:301-311 -- "layer,head,ratio" with the ratio printed "%.6f"."""
    r = np.asarray(ratios, np.float64).reshape(-1)
    if r.size != n_layers * n_kv_heads:
        raise ContractError("budget_table_csv: one ratio per (layer, kv head)")
    lines = ["layer,head,ratio"]
    lines += ["%d,%d,%.6f" % (l, h, r[l * n_kv_heads + h]) for l in range(n_layers) for h in range(n_kv_heads)]
    return "\n".join(lines) + "\n"


def budget_int_csv(budgets, n_layers: int, n_kv_heads: int) -> str:
    """tools/lkv.cpp:164-173 -- "layer,head,budget" with the frozen integer budgets."""
    b = np.asarray(budgets).reshape(-1)
    if b.size != n_layers * n_kv_heads:
        raise ContractError("budget_int_csv: one budget per (layer, kv head)")
    lines = ["layer,head,budget"]
    lines += ["%d,%d,%d" % (l, h, int(b[l * n_kv_heads + h])) for l in range(n_layers) for h in range(n_kv_heads)]
    return "\n".join(lines) + "\n"


def export_budgets(checkpoint: str, ratio: float, t: int, out_dir: str, device="cuda") -> tuple:
    """`lkv export-budgets` (tools/lkv.cpp:154-177) with the LKV-H solve and the freeze on the
    device (K2): writes budgets.csv (ratios) and, for t > 0, budgets_int.csv (floor budgets,
    freeze_budgets).  Returns the two paths (the second None when t <= 0)."""
    import os

    import torch

    from . import BUDGET_FLOOR, budgets as device_budgets

    p = load_lkv_params(checkpoint)
    logits = head_scores(p, device=device)
    ratios, b = device_budgets(logits, ratio, [max(int(t), 1)], BUDGET_FLOOR)
    os.makedirs(out_dir, exist_ok=True)
    p1 = os.path.join(out_dir, "budgets.csv")
    with open(p1, "w") as f:
        f.write(budget_table_csv(ratios.cpu().numpy(), p.n_layers, p.n_kv_heads))
    p2 = None
    if t > 0:
        p2 = os.path.join(out_dir, "budgets_int.csv")
        with open(p2, "w") as f:
            f.write(budget_int_csv(b[0].cpu().numpy(), p.n_layers, p.n_kv_heads))
    return p1, p2
