"""Times the C2 scorer (lkv_score, K1) and the fused eviction step; prints ms and GB/s."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_06676_b200 as lkv  # noqa: E402
from paper_2605_06676_b200 import synth  # noqa: E402

cfg = synth.CONFIGS[int(os.environ.get("CFG", "2"))]
cache = synth.make_cache(cfg)
sc = synth.make_scorers(cfg)
if os.environ.get("SCORER") == "ref":  # reference mode: [k;v] 2d -> d -> 1 SiLU, one scorer per (l, h)
    L, H, D = cfg.n_layers, cfg.n_kv_heads, cfg.head_dim
    g = torch.Generator(device="cuda").manual_seed(7)
    w1 = (torch.randn(L * H, 2 * D, D, generator=g, device="cuda") / (2 * D) ** 0.5).to(cfg.dtype)
    sc = lkv.Scorers(w1, torch.zeros(L * H, D, device="cuda"),
                     torch.randn(L * H, D, generator=g, device="cuda") / D ** 0.5,
                     input=lkv.SCORER_KV, activation=lkv.SILU, stride_layer=H, stride_head=1)
bpr = 4 + sc.input * cfg.head_dim * 2
ev = lkv.Evictor(cache, sc, synth.make_logits(cfg), cfg.ratio, lkv.BUDGET_EXACT)
out = torch.empty(cache.shape[:4], dtype=torch.float32, device="cuda")
cd, sd = cache.desc(), sc.desc()
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)


def score():
    lkv._check(lkv.lib().lkv_score(C.byref(cd), C.byref(sd), C.c_void_p(out.data_ptr()), None, 0, s))


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


ms_s = timeit(score)
ms_e = timeit(ev.launch)
ev.ws.status()
ref = lkv.token_scores(cache, sc)
rows = cache.n_heads * cache.shape[3]
print(f"score {ms_s:.4f} ms ({rows * bpr / ms_s / 1e6:.0f} GB/s)  evict {ms_e:.4f} ms  "
      f"check {float((out - ref).abs().max()):.2e}")
