"""Training-time operators of LKV on the B200.

* ``masked_attention_fwd`` / ``masked_attention_bwd`` -- the multiplicative soft-mask attention
  of ``attention.hpp:52-69`` (``masked_attention_dense`` + ``masked_attention_vjp``,
  ``attention.cpp:46-201``) for a batch of heads with GQA, i.e. every per-query-head call of
  ``forward_masked`` (``model.cpp:100-112``) in one launch; dK, dV and the mask gradient are
  summed over the query heads of a group, as the reference's autodiff accumulates them.
  Over the C ABI ``lkv_masked_attention_fwd`` / ``_bwd``.

Layouts: q / out / d_out ``[B, Hq, Tq, D]``; k / v ``[B, Hkv, Tk, D]`` (bf16 with D = 128 on
tensor cores, or fp32); mask ``[B, Hkv, Tk]`` fp32 or None; gradients fp32.
"""
from __future__ import annotations

import ctypes as C
import math

import torch

from . import ContractError, Workspace, _check, _dtype_code, _ptr, _stream, lib
from ._abi import AttnDesc


def _desc(q, k, causal, scale, pos_offset, self_keep) -> AttnDesc:
    if q.dim() != 4 or k.dim() != 4:
        raise ContractError("masked attention: q [B,Hq,Tq,D] and k/v [B,Hkv,Tk,D] required")
    B, Hq, Tq, D = q.shape
    Bk, Hkv, Tk, Dk = k.shape
    if Bk != B or Dk != D:
        raise ContractError("masked attention: q/k/v shape mismatch")
    scale = 1.0 / math.sqrt(D) if scale is None else float(scale)
    return AttnDesc(B, Hq, Hkv, Tq, Tk, D, _dtype_code(q.dtype), int(causal), int(pos_offset), int(self_keep), scale)


def _ws(desc: AttnDesc, device) -> Workspace:
    n = lib().lkv_attn_workspace_bytes(C.byref(desc))
    if n == 0:
        _check(lib().lkv_masked_attention_fwd(C.byref(desc), None, None, None, None, None, None, None, 0, None))
    return Workspace(n, device=device)


def masked_attention_fwd(q, k, v, mask=None, causal=True, scale=None, pos_offset=0, self_keep=False,
                         ws: Workspace | None = None, check=True):
    """-> (out [B,Hq,Tq,D] in q's dtype, lse [B,Hq,Tq] fp32, log2 domain)."""
    q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    if k.shape != v.shape or k.dtype != q.dtype or v.dtype != q.dtype:
        raise ContractError("masked attention: k/v must match and share q's dtype")
    desc = _desc(q, k, causal, scale, pos_offset, self_keep)
    m = mask.to(torch.float32).contiguous() if mask is not None else None
    if m is not None and tuple(m.shape) != tuple(k.shape[:3]):
        raise ContractError("masked attention: mask must be [B, Hkv, Tk]")
    ws = ws or _ws(desc, q.device)
    out = torch.empty_like(q)
    lse = torch.empty(q.shape[:3], dtype=torch.float32, device=q.device)
    _check(lib().lkv_masked_attention_fwd(C.byref(desc), _ptr(q), _ptr(k), _ptr(v), _ptr(m), _ptr(out), _ptr(lse),
                                          C.c_void_p(ws.ptr), ws.nbytes, _stream()))
    if check:
        ws.status()
    return out, lse


def masked_attention_bwd(q, k, v, mask, out, lse, d_out, causal=True, scale=None, pos_offset=0, self_keep=False,
                         ws: Workspace | None = None, check=True):
    """-> (dq [B,Hq,Tq,D], dk, dv [B,Hkv,Tk,D], dmask [B,Hkv,Tk] or None), all fp32."""
    q, k, v, d_out = q.contiguous(), k.contiguous(), v.contiguous(), d_out.contiguous().to(q.dtype)
    desc = _desc(q, k, causal, scale, pos_offset, self_keep)
    m = mask.to(torch.float32).contiguous() if mask is not None else None
    ws = ws or _ws(desc, q.device)
    dq = torch.empty(q.shape, dtype=torch.float32, device=q.device)
    dk = torch.empty(k.shape, dtype=torch.float32, device=q.device)
    dv = torch.empty(k.shape, dtype=torch.float32, device=q.device)
    dm = torch.empty(k.shape[:3], dtype=torch.float32, device=q.device) if m is not None else None
    out = out.contiguous()
    _check(lib().lkv_masked_attention_bwd(C.byref(desc), _ptr(q), _ptr(k), _ptr(v), _ptr(m), _ptr(out),
                                          _ptr(lse), _ptr(d_out), _ptr(dq), _ptr(dk), _ptr(dv), _ptr(dm),
                                          C.c_void_p(ws.ptr), ws.nbytes, _stream()))
    if check:
        ws.status()
    return dq, dk, dv, dm


# ---- Soft-TopK (soft_topk.hpp:60-67) -------------------------------------------------------------
def soft_topk(x, k, tau: float = 1.0, noise=None, noise_scale: float = 1.0, f32_mask: bool = False,
              ws: Workspace | None = None, check=True):
    """soft_topk_forward for every row of x [n_seg, n] (fp64) with budgets k [n_seg];
    scores are x + noise_scale * noise when noise is given (training_mask, policy.cpp:138-150).
    -> (values fp64, density fp64, lambda [n_seg], values_f32 or None)."""
    x = x.to(torch.float64).contiguous()
    if x.dim() == 1:
        x = x.view(1, -1)
    n_seg, n = x.shape
    kk = torch.as_tensor(k, dtype=torch.float64, device=x.device).reshape(-1).contiguous()
    if kk.numel() == 1 and n_seg > 1:
        kk = kk.expand(n_seg).contiguous()
    if kk.numel() != n_seg:
        raise ContractError("soft_topk: one budget per segment")
    nz = noise.to(torch.float64).contiguous().view(n_seg, n) if noise is not None else None
    vals = torch.empty_like(x)
    dens = torch.empty_like(x)
    lam = torch.empty(n_seg, dtype=torch.float64, device=x.device)
    v32 = torch.empty(n_seg, n, dtype=torch.float32, device=x.device) if f32_mask else None
    ws = ws or Workspace(256, device=x.device)
    _check(lib().lkv_soft_topk_fwd(_ptr(x), _ptr(nz), float(noise_scale), n_seg, n, n, _ptr(kk), float(tau),
                                   _ptr(vals), _ptr(dens), _ptr(v32), _ptr(lam), C.c_void_p(ws.ptr), ws.nbytes,
                                   _stream()))
    if check:
        ws.status()
    return vals, dens, lam, v32


def soft_topk_vjp(density, upstream, tau: float = 1.0):
    """soft_topk_vjp per segment -> (grad_x [n_seg, n], grad_k [n_seg])."""
    d = density.to(torch.float64).contiguous()
    if d.dim() == 1:
        d = d.view(1, -1)
    u = upstream.to(torch.float64).contiguous().view(d.shape)
    n_seg, n = d.shape
    gx = torch.empty_like(d)
    gk = torch.empty(n_seg, dtype=torch.float64, device=d.device)
    _check(lib().lkv_soft_topk_vjp(_ptr(d), _ptr(u), n_seg, n, n, float(tau), _ptr(gx), _ptr(gk), _stream()))
    return gx, gk
