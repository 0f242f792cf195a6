"""Minimal driver for ncu captures: the bench's C2 eviction step and decode steps.

    python profiles/step.py [--evict N] [--decode N] [--config 2]

Runs N fused eviction steps (lkv_evict through the C ABI) and N decode steps
over the resulting ragged cache; prints nothing but a final OK.  Used as
`<cmd>` in the recipes of /opt/skills/guides/B200_PROFILING.md.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2605_06676_b200 as lkv  # noqa: E402
from paper_2605_06676_b200 import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--evict", type=int, default=3)
ap.add_argument("--decode", type=int, default=3)
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--n-layers", type=int, default=0, help="fewer layers (e.g. one rank's share of a head-sharded run)")
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
cache = synth.make_cache(cfg, n_layers=a.n_layers or None)
L = a.n_layers or cfg.n_layers
ev = lkv.Evictor(cache, synth.make_scorers(cfg, n_layers=L), synth.make_logits(cfg, n_layers=L), cfg.ratio, lkv.BUDGET_EXACT,
                 decode_slack=a.decode + 8)
for _ in range(a.evict):
    ev.launch()
ev.ws.status()
rc = ev.ragged
rc.tokens_seen.copy_(torch.tensor(cache.seq_lens, dtype=torch.int32))
q, k, v = synth.make_decode_inputs(cfg, 0)
for _ in range(a.decode):
    lkv.decode_step(rc, q, k, v, check=False)
torch.cuda.synchronize()
if rc._decode_ws is not None:
    rc._decode_ws.status()
print("OK")
