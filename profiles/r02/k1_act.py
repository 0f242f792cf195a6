"""K1 (lkv_score, tcgen05) at C3 with the GELU-erf scorer vs the same weights under SiLU: is the
scorer epilogue on the critical path?"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2605_06676_b200 as lkv  # noqa: E402
from paper_2605_06676_b200 import synth  # noqa: E402

cfg = synth.CONFIGS[3]
cache = synth.make_cache(cfg)
g = synth.make_scorers(cfg)
out = torch.empty(cache.shape[:4], dtype=torch.float32, device="cuda")
cd = cache.desc()
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
res = {}
for name, act in (("gelu_erf", g.activation), ("silu", lkv.SILU)):
    sc = lkv.Scorers(g.w1, g.b1, g.w2, input=g.input, activation=act, stride_layer=g.stride_layer,
                     stride_head=g.stride_head)
    sd = sc.desc()

    def score():
        lkv._check(lkv.lib().lkv_score(C.byref(cd), C.byref(sd), C.c_void_p(out.data_ptr()), None, 0, s))

    for _ in range(3):
        score()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        score()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    rows = cache.keys.numel() // cfg.head_dim
    res[name] = {"ms": ms, "GB/s": rows * 260 / (ms / 1e3) / 1e9}
print(json.dumps(res))
