"""Layer-by-layer prefill with eviction at the C2 geometry.

    python profiles/prefill_time.py [--t 32768] [--reps 5]

Per layer (unfused form): the K/V projections (plain cuBLAS GEMMs x @ Wk, x @ Wv), then lkv_rope_pack (RoPE at absolute positions + token-major -> head-major) and the per-layer
score/select into the one global ragged cache.  Reports the eviction-side time per layer (rope_pack
+ score + select, device-timed), rope_pack alone with its HBM GB/s (algorithmic bytes: read the
two projections, write the two roped layers = 4 * T * H * D * 2 B), and the peak KV footprint
versus the full cache (the evictsim.cpp:157-159 accounting).  Fused form: hidden states ->
lkv_kv_project (K/V GEMM on CTA pairs with RoPE + pack in the epilogue) -> score/select, all 32
layers (ingest_layer_hidden), device-timed end to end.
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2605_06676_b200 as lkv  # noqa: E402
from paper_2605_06676_b200 import prefill, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--t", type=int, default=32768)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    cfg = synth.CONFIGS[2]
    L, H, D, T = cfg.n_layers, cfg.n_kv_heads, cfg.head_dim, a.t
    dm = cfg.n_q_heads * D
    g = torch.Generator(device="cuda").manual_seed(7)
    x = torch.randn(1, T, dm, generator=g, device="cuda").to(torch.bfloat16)
    wk = (torch.randn(dm, H * D, generator=g, device="cuda") / dm ** 0.5).to(torch.bfloat16)
    wv = (torch.randn(dm, H * D, generator=g, device="cuda") / dm ** 0.5).to(torch.bfloat16)
    scorers = synth.make_scorers(cfg)
    logits = synth.make_logits(cfg)
    k_lin = x @ wk
    v_lin = x @ wv
    pf = prefill.LayerwisePrefill(1, L, H, D, T, [T], scorers, logits, cfg.ratio, lkv.BUDGET_EXACT, decode_slack=4)
    for l in range(L):  # warm
        pf.ingest_layer(l, k_lin, v_lin)
    pf.finish()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    tot_gemm = tot_evict = 0.0
    for _ in range(a.reps):
        pf = prefill.LayerwisePrefill(1, L, H, D, T, [T], scorers, logits, cfg.ratio, lkv.BUDGET_EXACT,
                                      decode_slack=4)
        torch.cuda.synchronize()
        for l in range(L):
            ev[0].record()
            k_lin = x @ wk
            v_lin = x @ wv
            ev[1].record()
            pf.ingest_layer(l, k_lin, v_lin)
            ev[2].record()
            torch.cuda.synchronize()
            tot_gemm += ev[0].elapsed_time(ev[1])
            tot_evict += ev[1].elapsed_time(ev[2])
        pf.finish()
    n = a.reps * L
    # rope_pack alone
    tab = pf.table
    for _ in range(3):
        prefill.rope_pack(k_lin, v_lin, tab, [T], H)
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(20):
        prefill.rope_pack(k_lin, v_lin, tab, [T], H)
    ev[1].record()
    torch.cuda.synchronize()
    rp_ms = ev[0].elapsed_time(ev[1]) / 20
    rp_bytes = 4 * T * H * D * 2
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6545.9
    full_kv = L * H * T * D * 2 * 2
    # the fused path: hidden states -> lkv_kv_project (2-SM tcgen05 GEMM + RoPE + pack) -> score/select
    wkv_t = prefill.kv_weights(wk, wv)
    pf2 = prefill.LayerwisePrefill(1, L, H, D, T, [T], scorers, logits, cfg.ratio, lkv.BUDGET_EXACT, decode_slack=4)
    for l in range(L):  # warm
        pf2.ingest_layer_hidden(l, x, wkv_t)
    pf2.finish()
    tot_fused = 0.0
    for _ in range(a.reps):
        pf2 = prefill.LayerwisePrefill(1, L, H, D, T, [T], scorers, logits, cfg.ratio, lkv.BUDGET_EXACT,
                                       decode_slack=4)
        torch.cuda.synchronize()
        ev[0].record()
        for l in range(L):
            pf2.ingest_layer_hidden(l, x, wkv_t)
        ev[1].record()
        torch.cuda.synchronize()
        tot_fused += ev[0].elapsed_time(ev[1])
        pf2.finish()
    assert torch.equal(pf2.ragged.lens, pf.ragged.lens)
    print(json.dumps({
        "fused_prefill_ms_all_layers": tot_fused / a.reps,
        "fused_prefill_ms_per_layer": tot_fused / a.reps / L,
        "unfused_ms_all_layers": (tot_gemm + tot_evict) / a.reps,
        "what": "layer-by-layer prefill eviction, C2 geometry (L32 H8 d128), bf16, R=0.15",
        "t": T, "evict_ms_per_layer": tot_evict / n, "evict_ms_all_layers": tot_evict / a.reps,
        "kv_gemms_ms_per_layer": tot_gemm / n,
        "rows_per_s": L * H * T / (tot_evict / a.reps / 1e3),
        "rope_pack_ms": rp_ms, "rope_pack_gbs": rp_bytes / (rp_ms / 1e3) / 1e9,
        "rope_pack_frac_of_measured_hbm": rp_bytes / (rp_ms / 1e3) / 1e9 / peak,
        "peak_kv_bytes": pf.peak_kv_bytes, "full_kv_bytes": full_kv,
        "peak_over_full": pf.peak_kv_bytes / full_kv}))


if __name__ == "__main__":
    main()
