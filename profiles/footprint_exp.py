"""Experiment: does the scorer's bandwidth depend on the cache footprint one launch spans?
Times lkv_score on the whole C5 cache, per sequence, and per (sequence, layer-group)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_06676_b200 as lkv  # noqa: E402
from paper_2605_06676_b200 import synth  # noqa: E402

cfg = synth.CONFIGS[int(os.environ.get("CFG", "5"))]
cache = synth.make_cache(cfg)
if os.environ.get("UNIFORM"):
    cache = lkv.DenseCache(cache.keys, cache.values, [int(os.environ["UNIFORM"])] * cache.shape[0])
sc = synth.make_scorers(cfg)
S, L, H, T, D = cache.shape
out = torch.empty(S, L, H, T, dtype=torch.float32, device="cuda")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
lib = lkv.lib()


def run_parts(lg):
    descs = []
    for s in range(S):
        for l0 in range(0, L, lg):
            k = cache.keys[s:s + 1, l0:l0 + lg]
            v = cache.values[s:s + 1, l0:l0 + lg]
            sub = lkv.DenseCache(k, v, [cache.seq_lens[s]])
            w1 = sc.w1[l0:l0 + lg]
            sub_sc = lkv.Scorers(w1, sc.b1[l0:l0 + lg], sc.w2[l0:l0 + lg], input=sc.input, activation=sc.activation)
            o = out[s:s + 1, l0:l0 + lg]
            descs.append((sub, sub_sc, sub.desc(), sub_sc.desc(), o))

    def fn():
        for sub, sub_sc, cd, sd, o in descs:
            lkv._check(lib.lkv_score(C.byref(cd), C.byref(sd), C.c_void_p(o.data_ptr()), None, 0, st))
    return fn


def timeit(fn, n=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


rows = sum(cache.seq_lens) * L * H
cd, sd = cache.desc(), sc.desc()
full = lambda: lkv._check(lib.lkv_score(C.byref(cd), C.byref(sd), C.c_void_p(out.data_ptr()), None, 0, st))  # noqa
for name, fn in [("whole cache", full), ("per sequence", run_parts(L)), ("per 8 layers", run_parts(8)),
                 ("per 4 layers", run_parts(4))]:
    ms = timeit(fn)
    print(f"{name:14s} {ms:.3f} ms  {rows * 260 / ms / 1e6:.0f} GB/s")
