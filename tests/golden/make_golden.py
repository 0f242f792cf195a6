"""Regenerates the committed policy-checkpoint fixtures with the reference's OWN code
(oracle/_ref: the unmodified proj/src/policy.cpp init + checkpoint.cpp/container.cpp save,
compiled from /root/reference).  Run here (where /root/reference exists):

    python tests/golden/make_golden.py

Outputs (small, committed): lkv_params_desk.bin (the reference's default ModelConfig:
4 layers x 2 KV heads, d=16, d_e=16) and lkv_params_l2h4d128.bin (2 x 4, d=128, d_e=32),
plus their LKV-H logits from the reference's own load_lkv_params + head_scores.
"""
import ctypes as C
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle as O  # noqa: E402

CASES = {"desk": (4, 2, 16, 16, 7), "l2h4d128": (2, 4, 128, 32, 11)}


def main():
    O.build()
    ref = O.ref_lib()
    assert ref is not None, "needs /root/reference (oracle/_ref)"
    ref.ref_write_lkv_params.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_ulonglong]
    ref.ref_head_scores.argtypes = [C.c_char_p, C.POINTER(C.c_double), C.c_int]
    for name, (L, H, d, de, seed) in CASES.items():
        path = os.path.join(HERE, f"lkv_params_{name}.bin")
        assert ref.ref_write_lkv_params(path.encode(), L, H, d, de, seed) == 0
        logits = np.empty(L * H)
        assert ref.ref_head_scores(path.encode(), logits.ctypes.data_as(C.POINTER(C.c_double)), L * H) == 0
        np.save(os.path.join(HERE, f"head_scores_{name}.npy"), logits)
        print(path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
