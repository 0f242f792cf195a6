"""Relative gradient error (max|gpu - oracle| / max|oracle|) of the bf16 masked-attention backward
over several seeds and lengths (the fp64 oracle on the same bf16-rounded inputs).

    python profiles/attn_grad_error.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from test_train_gpu import _inputs, _oracle, rel_gap  # noqa: E402
from paper_2605_06676_b200 import train  # noqa: E402

for T in (640, 1536):
    gaps = {k: [] for k in ("out", "dq", "dk", "dv", "dmask")}
    for seed in range(6):
        q, k, v, du, mask = _inputs(1, 4, 1, T, T, 128, torch.bfloat16, True, seed)
        scale = 1.0 / np.sqrt(128)
        out, lse = train.masked_attention_fwd(q, k, v, mask, True, scale, 0, False)
        got = [out, *train.masked_attention_bwd(q, k, v, mask, out, lse, du, True, scale, 0, False)]
        ref = _oracle(q, k, v, mask, du, True, scale, 0, False)
        for name, g_, r in zip(gaps, got, ref):
            gaps[name].append(rel_gap(g_.double().cpu().numpy(), r))
    print(T, {k: (round(min(v), 4), round(max(v), 4)) for k, v in gaps.items()})
