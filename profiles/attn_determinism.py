"""Repeat the masked-attention forward / backward on identical inputs and count runs whose
outputs differ bitwise from the first (every kernel is meant to be deterministic).

    python profiles/attn_determinism.py [--t 640] [--reps 50]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_06676_b200 import train  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--t", type=int, default=640)
ap.add_argument("--reps", type=int, default=50)
ap.add_argument("--hq", type=int, default=4)
ap.add_argument("--hkv", type=int, default=1)
a = ap.parse_args()
g = torch.Generator(device="cuda").manual_seed(3)
B, Hq, Hkv, T, D = 1, a.hq, a.hkv, a.t, 128
q = torch.randn(B, Hq, T, D, generator=g, device="cuda").to(torch.bfloat16)
k = torch.randn(B, Hkv, T, D, generator=g, device="cuda").to(torch.bfloat16)
v = torch.randn(B, Hkv, T, D, generator=g, device="cuda").to(torch.bfloat16)
du = torch.randn(B, Hq, T, D, generator=g, device="cuda").to(torch.bfloat16)
m = torch.rand(B, Hkv, T, generator=g, device="cuda")
m[:, :, 0] = 1.0
out0, lse0 = train.masked_attention_fwd(q, k, v, m)
ref = train.masked_attention_bwd(q, k, v, m, out0, lse0, du)
bad = {"out": 0, "lse": 0, "dq": 0, "dk": 0, "dv": 0, "dmask": 0}
for _ in range(a.reps):
    out, lse = train.masked_attention_fwd(q, k, v, m)
    bad["out"] += int(not torch.equal(out, out0))
    bad["lse"] += int(not torch.equal(lse, lse0))
    got = train.masked_attention_bwd(q, k, v, m, out0, lse0, du)
    for name, x, y in zip(["dq", "dk", "dv", "dmask"], got, ref):
        bad[name] += int(not torch.equal(x, y))
print({"T": T, "reps": a.reps, "runs_differing": bad})
