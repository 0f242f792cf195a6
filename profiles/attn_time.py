"""Timing of the training-time masked attention at Llama-3-8B head geometry.

    python profiles/attn_time.py [--t 4096] [--b 1]

Hq = 32, Hkv = 8, d = 128, bf16, causal, a random soft mask.  Reports forward and backward
ms and tensor TFLOP/s (algorithmic flops of the causal triangle: fwd 2 GEMMs, bwd 5 GEMMs,
i.e. what a one-pass backward must do; the two-kernel backward recomputes S and dP once more).
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_06676_b200 import train  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--t", type=int, default=4096)
    ap.add_argument("--b", type=int, default=1)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--nocheck", action="store_true", help="skip device error checks (bisection builds)")
    a = ap.parse_args()
    B, Hq, Hkv, T, D = a.b, 32, 8, a.t, 128
    g = torch.Generator(device="cuda").manual_seed(0)
    q = torch.randn(B, Hq, T, D, generator=g, device="cuda").to(torch.bfloat16)
    k = torch.randn(B, Hkv, T, D, generator=g, device="cuda").to(torch.bfloat16)
    v = torch.randn(B, Hkv, T, D, generator=g, device="cuda").to(torch.bfloat16)
    du = torch.randn(B, Hq, T, D, generator=g, device="cuda").to(torch.bfloat16)
    mask = torch.rand(B, Hkv, T, generator=g, device="cuda")
    out, lse = train.masked_attention_fwd(q, k, v, mask, check=not a.nocheck)
    train.masked_attention_bwd(q, k, v, mask, out, lse, du, check=not a.nocheck)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    torch.cuda.synchronize()
    e[0].record()
    for _ in range(a.reps):
        out, lse = train.masked_attention_fwd(q, k, v, mask, check=False)
    e[1].record()
    for _ in range(a.reps):
        train.masked_attention_bwd(q, k, v, mask, out, lse, du, check=False)
    e[2].record()
    torch.cuda.synchronize()
    fwd = e[0].elapsed_time(e[1]) / a.reps
    bwd = e[1].elapsed_time(e[2]) / a.reps
    tri = B * Hq * (T * (T + 1) / 2) * D  # causal multiply-adds per GEMM
    peak = 1676.6
    try:
        peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                           "MEASURED_PEAKS.json")))["bf16_tflops"]
    except Exception:
        pass
    # Soft-TopK over every (layer, kv head) token row of a C2-sized cache (training_mask)
    ns, nt = 256, a.t
    x = torch.randn(ns, nt, dtype=torch.float64, device="cuda", generator=g)
    kb = torch.full((ns,), 0.15 * nt, dtype=torch.float64, device="cuda")
    vals, dens, _, _ = train.soft_topk(x, kb, check=not a.nocheck)
    up = torch.randn_like(x)
    train.soft_topk_vjp(dens, up)
    torch.cuda.synchronize()
    e[0].record()
    for _ in range(a.reps):
        vals, dens, _, _ = train.soft_topk(x, kb, check=False)
    e[1].record()
    for _ in range(a.reps):
        train.soft_topk_vjp(dens, up)
    e[2].record()
    torch.cuda.synchronize()
    stk_f = e[0].elapsed_time(e[1]) / a.reps
    stk_b = e[1].elapsed_time(e[2]) / a.reps
    print(json.dumps({"what": "soft-topk fwd/vjp, 256 segments (L32 x H8) x t tokens, fp64", "t": nt,
                      "fwd_ms": stk_f, "vjp_ms": stk_b, "rows_per_s": ns * nt / (stk_f / 1e3)}))
    print(json.dumps({"what": "masked attention train, Llama-3-8B heads (32q/8kv, d128), causal, bf16", "B": B, "T": T,
                      "fwd_ms": fwd, "bwd_ms": bwd, "fwd_tflops": 2 * 2 * tri / fwd / 1e9,
                      "bwd_tflops": 5 * 2 * tri / bwd / 1e9, "bf16_peak_tflops": peak,
                      "fwd_frac": 2 * 2 * tri / fwd / 1e9 / peak, "bwd_frac": 5 * 2 * tri / bwd / 1e9 / peak}))


if __name__ == "__main__":
    main()
