"""Times 64 C2 decode steps (all layers per launch) after one eviction; prints ms/step and GB/s."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_06676_b200 as lkv  # noqa: E402
from paper_2605_06676_b200 import synth  # noqa: E402

cfg = synth.CONFIGS[int(os.environ.get("CFG", "2"))]
cache = synth.make_cache(cfg)
ev = lkv.Evictor(cache, synth.make_scorers(cfg), synth.make_logits(cfg), cfg.ratio, lkv.BUDGET_EXACT, decode_slack=80)
res = ev.run()
rc = res.cache
q, k, v = synth.make_decode_inputs(cfg, 0)
out = torch.empty_like(q)
for _ in range(3):
    lkv.decode_step(rc, q, k, v, out=out, check=False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 64
rows = int(rc.lens.sum()) + rc.n_heads * n // 2
e0.record()
for _ in range(n):
    lkv.decode_step(rc, q, k, v, out=out, check=False)
e1.record()
torch.cuda.synchronize()
rc._decode_ws.status()
ms = e0.elapsed_time(e1) / n
print(f"{ms:.4f} ms/step  {rows * 2 * 256 / ms / 1e6:.0f} GB/s")
