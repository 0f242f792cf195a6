"""Trained-policy ingestion: the reference's own checkpoint files (tests/golden, written by
the unmodified reference save path via tests/golden/make_golden.py) -> LKV-H logits and
LKV-T scorer tables for the device path."""
import os
import struct

import numpy as np
import pytest
import torch

import oracle as O
import paper_2605_06676_b200 as lkv
from paper_2605_06676_b200 import policy_io

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("name,L,H,d,de", [("desk", 4, 2, 16, 16), ("l2h4d128", 2, 4, 128, 32)])
def test_load_reference_checkpoint(name, L, H, d, de):
    p = policy_io.load_lkv_params(os.path.join(G, f"lkv_params_{name}.bin"))
    assert (p.n_layers, p.n_kv_heads, p.d_head, p.d_e) == (L, H, d, de)
    assert len(p.token_scorers) == L * H
    assert p.head_embeddings.shape == (L * H, de)
    assert p.head_predictor.w1.shape == (de, de // 2)
    # init_mlp2 (policy.cpp:18-28): b1 = 0, w1 ~ N(0, 1/in)
    assert all((m.b1 == 0).all() for m in p.token_scorers)
    assert abs(np.std(np.concatenate([m.w1.ravel() for m in p.token_scorers])) - 1 / np.sqrt(2 * d)) < 0.1 / np.sqrt(d)
    # the oracle's mlp2 on the loaded tables equals the reference's own load_lkv_params + head_scores
    want = np.load(os.path.join(G, f"head_scores_{name}.npy"))
    got = O.token_scores(p.head_embeddings, None, p.head_predictor.w1, p.head_predictor.b1, p.head_predictor.w2, act=O.SILU, dtype=O.F64)
    assert np.max(np.abs(got - want)) <= 1e-12 * max(1.0, np.max(np.abs(want)))
    # parameter count fixture (policy.cpp:289-299): 2d*d + d + d per scorer
    assert sum(m.w1.size + m.b1.size + m.w2.size for m in p.token_scorers) == L * H * (2 * d * d + 2 * d)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["desk", "l2h4d128"])
def test_device_head_scores_are_the_references(name):
    """The LKV-H logits computed on the B200 (fp64) equal the reference's own head_scores."""
    p = policy_io.load_lkv_params(os.path.join(G, f"lkv_params_{name}.bin"))
    want = np.load(os.path.join(G, f"head_scores_{name}.npy"))
    got = policy_io.head_scores(p).cpu().numpy()
    assert np.max(np.abs(got - want)) <= 1e-12 * max(1.0, np.max(np.abs(want)))
    r = O.allocate_budgets(got, 0.15)
    assert np.allclose(r, O.allocate_budgets(want, 0.15), rtol=1e-12, atol=0)


def test_container_validation(tmp_path):
    src = open(os.path.join(G, "lkv_params_desk.bin"), "rb").read()
    bad = tmp_path / "trunc.bin"
    bad.write_bytes(src[:4])
    with pytest.raises(lkv.ContractError):
        policy_io.load_container(str(bad))
    bad.write_bytes(src[:-3])
    with pytest.raises(lkv.ContractError):
        policy_io.load_container(str(bad))
    bad.write_bytes(src + b"xx")
    with pytest.raises(lkv.ContractError):
        policy_io.load_container(str(bad))
    (meta_len,) = struct.unpack("<Q", src[:8])
    bad.write_bytes(struct.pack("<Q", meta_len) + b"{" * meta_len + src[8 + meta_len:])
    with pytest.raises(lkv.ContractError):
        policy_io.load_container(str(bad))


@pytest.mark.gpu
def test_evict_with_reference_checkpoint():
    """Real LKV-H logits and LKV-T scorers from the reference checkpoint drive the device
    path (reference mode: [k;v] 256 -> 128 -> 1 SiLU per (l,h), floor budgets)."""
    p = policy_io.load_lkv_params(os.path.join(G, "lkv_params_l2h4d128.bin"))
    logits = torch.tensor(np.load(os.path.join(G, "head_scores_l2h4d128.npy")), device="cuda")
    torch.manual_seed(31)
    L, H, T, D = p.n_layers, p.n_kv_heads, 3000, p.d_head
    K = torch.randn(1, L, H, T, D, device="cuda").to(torch.bfloat16)
    V = torch.randn(1, L, H, T, D, device="cuda").to(torch.bfloat16)
    cache = lkv.DenseCache(K, V, [T])
    scorers = policy_io.scorers_from_params(p)
    res = lkv.evict(cache, scorers, logits, 0.15, lkv.BUDGET_FLOOR, keep_scores=True)
    want_b = O.freeze_budgets(O.allocate_budgets(logits.cpu().numpy(), 0.15), T)
    assert (res.budgets[0].cpu().numpy() == want_b).all()
    Kn = K.view(torch.int16).cpu().numpy().view(np.uint16)
    Vn = V.view(torch.int16).cpu().numpy().view(np.uint16)
    sc = res.scores.reshape(L * H, T).cpu().numpy()
    for h in range(L * H):
        l, kh = divmod(h, H)
        m = p.token_scorers[h]
        w1 = scorers.w1[h].double().cpu().numpy()  # bf16-rounded, as on the device
        ref = O.token_scores(Kn[0, l, kh], Vn[0, l, kh], w1, m.b1, m.w2, act=O.SILU)
        assert np.max(np.abs(sc[h] - ref)) / np.max(np.abs(ref)) <= 1e-2
        _, _, pos = res.cache.head(h)
        assert (pos.cpu().numpy() == O.select_positions_f32(sc[h], int(want_b[h]))).all()


def _ref_csv(scores, L, H, ratio):
    import ctypes as C

    R = O.ref_lib()
    R.ref_budget_table_csv.argtypes = [C.POINTER(C.c_double), C.c_int, C.c_int, C.c_double, C.c_char_p, C.c_int]
    x = np.ascontiguousarray(scores, np.float64)
    buf = C.create_string_buffer(1 << 20)
    assert R.ref_budget_table_csv(x.ctypes.data_as(C.POINTER(C.c_double)), L, H, ratio, buf, 1 << 20) == 0
    return buf.value.decode()


@pytest.mark.skipif(O.ref_lib() is None, reason="oracle/_ref not built (reference not mounted)")
def test_budget_csv_equals_the_references():
    """budget_table_csv (policy.cpp:301-311) byte-identical to the reference's own function."""
    rng = np.random.default_rng(8)
    for L, H, r in ((2, 4, 0.15), (32, 8, 0.1), (80, 8, 0.25)):
        x = rng.normal(0, 1.5, L * H)
        assert policy_io.budget_table_csv(O.allocate_budgets(x, r), L, H) == _ref_csv(x, L, H, r)


def test_budget_int_csv_format():
    """tools/lkv.cpp:164-173: header then one "l,h,budget" line per (layer, kv head)."""
    assert policy_io.budget_int_csv([150, 150, 3, 0], 2, 2) == "layer,head,budget\n0,0,150\n0,1,150\n1,0,3\n1,1,0\n"
    with pytest.raises(lkv.ContractError):
        policy_io.budget_int_csv([1, 2, 3], 2, 2)


@pytest.mark.gpu
def test_export_budgets_from_reference_checkpoint(tmp_path):
    """`lkv export-budgets` (tools/lkv.cpp:154-177) with the LKV-H solve on the device: the CSVs
    equal the reference's (ratios through its own budget_table_csv, floor budgets bit-exact)."""
    ck = os.path.join(G, "lkv_params_l2h4d128.bin")
    p1, p2 = policy_io.export_budgets(ck, 0.15, 1000, str(tmp_path))
    p = policy_io.load_lkv_params(ck)
    scores = policy_io.head_scores(p).cpu().numpy()
    want_ratios = O.allocate_budgets(scores, 0.15)
    assert open(p1).read() == policy_io.budget_table_csv(want_ratios, p.n_layers, p.n_kv_heads)
    if O.ref_lib() is not None:
        assert open(p1).read() == _ref_csv(scores, p.n_layers, p.n_kv_heads, 0.15)
    assert open(p2).read() == policy_io.budget_int_csv(O.freeze_budgets(want_ratios, 1000), p.n_layers, p.n_kv_heads)
