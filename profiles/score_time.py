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
print(f"score {ms_s:.4f} ms ({rows * 260 / ms_s / 1e6:.0f} GB/s)  evict {ms_e:.4f} ms  "
      f"check {float((out - ref).abs().max()):.2e}")
