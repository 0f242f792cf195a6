"""K/V production for layer-by-layer prefill at the C2 layer geometry (T tokens x d_model 4096 ->
8 KV heads x 128 for K and V): lkv_kv_project (tcgen05 GEMM, RoPE + head-major pack fused in the
epilogue) against the unfused path it replaces (cuBLAS x @ [Wk | Wv] via torch, then lkv_rope_pack).

    python profiles/kvproj_time.py [--t 32768] [--reps 20]

Prints one JSON line: ms per layer for each path, TFLOP/s of the fused kernel against the measured
dense bf16 peak (MEASURED_PEAKS.json), and the fused/unfused ratio."""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2605_06676_b200 import prefill  # noqa: E402


def timed(fn, reps):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--t", type=int, default=32768)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    T, H, D, dm = a.t, 8, 128, 4096
    g = torch.Generator(device="cuda").manual_seed(7)
    h = torch.randn(1, T, dm, generator=g, device="cuda").to(torch.bfloat16)
    wk = (torch.randn(dm, H * D, generator=g, device="cuda") / dm ** 0.5).to(torch.bfloat16)
    wv = (torch.randn(dm, H * D, generator=g, device="cuda") / dm ** 0.5).to(torch.bfloat16)
    w = torch.cat([wk, wv], dim=1)
    wt = prefill.kv_weights(wk, wv)
    tab = prefill.rope_table(T, D)
    k_out = torch.empty(1, 1, H, T, D, dtype=torch.bfloat16, device="cuda")
    v_out = torch.empty_like(k_out)

    def fused():
        prefill.kv_project(h, wt, tab, [T], H)

    def unfused():
        kv = h @ w
        prefill.rope_pack(kv[..., :H * D], kv[..., H * D:], tab, [T], H)

    def gemm_only():
        h @ w

    t_f, t_u, t_g = timed(fused, a.reps), timed(unfused, a.reps), timed(gemm_only, a.reps)
    # agreement of the two paths (the unfused one rounds the projection to bf16 before RoPE)
    kf, vf = prefill.kv_project(h, wt, tab, [T], H)
    kv = h @ w
    ku, vu = prefill.rope_pack(kv[..., :H * D], kv[..., H * D:], tab, [T], H)
    gap = float((kf.float() - ku.float()).abs().max() / ku.float().abs().max())
    gap_v = float((vf.float() - vu.float()).abs().max() / vu.float().abs().max())
    # both against fp64 on sampled rows (positions spread over the whole sequence)
    import numpy as np

    rows = [0, 1, 777, T // 2 + 3, T - 1]
    hd = h[0, rows].double().cpu().numpy()
    kl = (hd @ wk.double().cpu().numpy()).reshape(len(rows), H, D)
    th = np.array(rows)[:, None] * (10000.0 ** (-2.0 * np.arange(D // 2) / D))[None, :]
    want = np.empty_like(kl)
    a_, b_ = kl[..., 0::2], kl[..., 1::2]
    want[..., 0::2] = a_ * np.cos(th)[:, None, :] - b_ * np.sin(th)[:, None, :]
    want[..., 1::2] = a_ * np.sin(th)[:, None, :] + b_ * np.cos(th)[:, None, :]
    fused_k = kf[0, 0][:, rows].double().cpu().numpy().transpose(1, 0, 2)
    unfused_k = ku[0, 0][:, rows].double().cpu().numpy().transpose(1, 0, 2)
    gap_fused = float(np.abs(fused_k - want).max() / np.abs(want).max())
    gap_unfused = float(np.abs(unfused_k - want).max() / np.abs(want).max())
    flops = 2.0 * T * dm * 2 * H * D
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"]
    except Exception:
        peak = 1590.0
    print(json.dumps({"what": "K/V projection per layer, C2 geometry", "t": T, "d_model": dm, "n_kv_heads": H,
                      "fused_ms": t_f, "fused_tflops": flops / t_f / 1e9, "fused_frac_of_measured_bf16":
                      flops / t_f / 1e9 / peak, "cublas_gemm_ms": t_g, "cublas_tflops": flops / t_g / 1e9,
                      "unfused_ms": t_u, "speedup_vs_unfused": t_u / t_f, "rel_gap_vs_unfused_k": gap, "fused_k_gap_vs_fp64": gap_fused, "unfused_k_gap_vs_fp64": gap_unfused,
                      "rel_gap_vs_unfused_v": gap_v}))


if __name__ == "__main__":
    main()
