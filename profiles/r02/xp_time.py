"""Times K1 alone (lkv_score) and the fused step (lkv_evict) at C3 with the library in place:
    python profiles/r02/xp_time.py [reps]"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2605_06676_b200 as lkv  # noqa: E402
from paper_2605_06676_b200 import synth  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
cfg = synth.CONFIGS[3]
cache = synth.make_cache(cfg)
ev = lkv.Evictor(cache, synth.make_scorers(cfg), synth.make_logits(cfg), cfg.ratio, lkv.BUDGET_EXACT, decode_slack=8)
L = lkv.lib()
sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
scores = torch.empty(cache.n_heads * cfg.max_tokens, dtype=torch.float32, device="cuda")


def score():
    lkv._check(L.lkv_score(C.byref(ev._cd), C.byref(ev._sd), C.c_void_p(scores.data_ptr()), None, 0, sp))


def timed(fn):
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


out = {"score_ms": timed(score), "step_ms": timed(ev.launch)}
ev.ws.status()
out["score_ms_2"] = timed(score)
print(json.dumps(out))
