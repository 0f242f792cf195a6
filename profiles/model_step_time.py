"""Full decode step at Llama-3-8B geometry over an evicted C2 cache.

    python profiles/model_step_time.py [--n-seq 1] [--steps 50] [--vocab 128256]

Random bf16 weights (N(0, 0.02)) in the reference's parameter layout, a C2 cache (t = 32768,
R = 0.15) evicted by lkv_evict, then `steps` decode steps replayed from a CUDA graph.  Reports
ms/step and the HBM bytes a step must read (every weight once + every retained K/V row) against
the measured copy peak -- decode is weight-streaming, so that fraction is the roofline.
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2605_06676_b200 as lkv  # noqa: E402
from paper_2605_06676_b200 import model as M, synth  # noqa: E402


def trace_replay(g, path):
    """One replay with the experiment build's per-CTA (kind, entry, wait released, exit) records."""
    import ctypes
    import numpy as np
    lib = ctypes.CDLL(lkv._abi.LIB_PATH)
    lib.lkv_xp_trace.restype = ctypes.c_int32
    lib.lkv_xp_trace(None, 0)
    g.replay()
    torch.cuda.synchronize()
    rec = np.zeros(1 << 20, dtype=[("kind", "<u4"), ("cta", "<u4")] + [(f"t{i}", "<u8") for i in range(6)])
    n = lib.lkv_xp_trace(rec.ctypes.data_as(ctypes.c_void_p), 1 << 20)
    np.save(path, rec[:n])
    print("trace records", n)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-seq", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--vocab", type=int, default=128256)
    ap.add_argument("--t", type=int, default=32768)
    ap.add_argument("--eager", action="store_true", help="eager steps, no graph (for ncu launch lists)")
    ap.add_argument("--trace", default="",
                    help="experiment builds with LKV_XP_TRACE: write one replay's per-CTA timeline here")
    ap.add_argument("--rows-per-item", type=int, default=0,
                    help="per-layer attention work-item rows (0: the one-wave plan)")
    a = ap.parse_args()
    torch.manual_seed(0)
    cfg = M.ModelConfig(n_layers=32, n_query_heads=32, n_kv_heads=8, head_dim=128, vocab_size=a.vocab,
                        max_seq_len=a.t + a.steps + 64, mlp_hidden=14336)
    dm, dkv, ff = cfg.d_model, cfg.n_kv_heads * cfg.head_dim, cfg.mlp_width
    shapes = {"wq": (dm, dm), "wk": (dm, dkv), "wv": (dm, dkv), "wo": (dm, dm), "attn_norm": (dm,),
              "mlp_norm": (dm,), "w_gate": (dm, ff), "w_up": (dm, ff), "w_down": (ff, dm)}
    params = {}
    for name in M.param_names(cfg):
        if name == "tok_embed":
            shp = (cfg.vocab_size, dm)
        elif name == "final_norm":
            shp = (dm,)
        elif name == "lm_head":
            shp = (dm, cfg.vocab_size)
        else:
            shp = shapes[name.split(".")[2]]
        if len(shp) == 1:
            params[name] = torch.ones(shp, dtype=torch.bfloat16, device="cuda")
        else:
            params[name] = (torch.randn(shp, device="cuda") * 0.02).to(torch.bfloat16)
    model = M.DecodeModel(cfg, params)
    w_bytes = sum(int(v.numel()) * 2 for k, v in params.items() if k != "tok_embed")
    del params
    torch.cuda.empty_cache()
    c2 = synth.CONFIGS[2]
    cache = synth.make_cache(c2, n_seq=a.n_seq, max_tokens=a.t)
    res = lkv.evict(cache, synth.make_scorers(c2), synth.make_logits(c2), c2.ratio, lkv.BUDGET_EXACT,
                    decode_slack=a.steps + 8, keep_scores=False)
    del cache
    torch.cuda.empty_cache()
    rc = res.cache
    model.bind(rc, rows_per_item=a.rows_per_item)
    tokens = torch.randint(0, cfg.vocab_size, (a.n_seq,), dtype=torch.int32, device="cuda")
    logits = torch.empty(a.n_seq, cfg.vocab_size, dtype=torch.float32, device="cuda")
    model.step(tokens, logits)  # eager step, error-checked
    if a.eager:
        for _ in range(a.steps):
            model.step(tokens, logits, check=False)
        torch.cuda.synchronize()
        model.ws.status()
        print("eager steps done")
        return
    g = model.capture(tokens, logits)
    lens0 = rc.lens.clone()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    model.ws.status()
    ms = e0.elapsed_time(e1) / a.steps
    if a.trace:
        trace_replay(g, a.trace)
    kv_rows = float(lens0.double().sum()) + 1.5 * a.steps * rc.n_heads + 3 * rc.n_heads
    kv_bytes = kv_rows * 2 * cfg.head_dim * 2
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6545.9
    gbs = (w_bytes + kv_bytes) / (ms / 1e3) / 1e9
    print(json.dumps({"what": "full decode step, Llama-3-8B geometry, bf16, CUDA graph", "n_seq": a.n_seq,
                      "vocab": cfg.vocab_size, "cache": f"C2 t={a.t} R=0.15 evicted", "ms_per_step": ms,
                      "tokens_per_s": a.n_seq / (ms / 1e3), "weight_bytes": w_bytes, "kv_bytes_per_step": kv_bytes,
                      "hbm_gbs": gbs, "frac_of_measured_hbm": gbs / peak}))


if __name__ == "__main__":
    main()
