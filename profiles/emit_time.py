"""Times the C2 select (+fused gather) stage alone on precomputed scores/budgets."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_06676_b200 as lkv  # noqa: E402
from paper_2605_06676_b200 import synth  # noqa: E402

cfg = synth.CONFIGS[int(os.environ.get("CFG", "2"))]
cache = synth.make_cache(cfg)
ev = lkv.Evictor(cache, synth.make_scorers(cfg), synth.make_logits(cfg), cfg.ratio, lkv.BUDGET_EXACT,
                 keep_scores=True)
ev.run()
lib = lkv.lib()
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
cd, rd = ev._cd, ev._rd


def sel():
    lkv._check(lib.lkv_select(C.byref(cd), C.c_void_p(ev.scores.data_ptr()), C.c_void_p(ev.budgets.data_ptr()),
                              C.byref(rd), 1, C.c_void_p(ev.ws.ptr), ev.ws.nbytes, st))


for _ in range(3):
    sel()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 20
e0.record()
for _ in range(n):
    sel()
e1.record()
torch.cuda.synchronize()
ev.ws.status()
ms = e0.elapsed_time(e1) / n
kept = int(ev.ragged.lens.sum())
moved = kept * 2 * 2 * cfg.head_dim * 2
print(f"select+gather {ms:.4f} ms  gather {moved / ms / 1e6:.0f} GB/s (read+write)")
