"""CPU oracle for LKV's inference-time eviction path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import this package, and only as the checker or as
the reported CPU baseline.  The product (``paper_2605_06676_b200``) never imports
it and has no CPU fallback.

Two libraries back it:

* ``oracle/liblkv_oracle.so`` -- the fp64 plain-C restatement (``lkv_oracle.c``),
  each function citing the reference file:line it follows;
* ``oracle/_ref/liblkv_ref.so`` (optional) -- the reference's own
  ``proj/src/{tensor,attention,model,soft_topk,policy,evictsim,...}.cpp`` compiled
  unmodified from ``/root/reference`` (Eigen, absent here, replaced by our own minimal
  compat header ``oracle/ref_shim/eigen``), used to pin the restatement.  Built only
  where ``/root/reference`` exists.
* ``oracle/model.py`` -- fp64 numpy restatement of the toy model's decode step.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liblkv_oracle.so")
_REF_PATH = os.path.join(_HERE, "_ref", "liblkv_ref.so")
# the same source built like the reference builds itself (-O3, AVX2/FMA): the CPU-baseline timer only
_FAST_PATH = os.path.join(_HERE, "liblkv_oracle_fast.so")

OK, CONTRACT, NUMERIC, BUDGET, OVERFLOW_GUARD, DEGENERATE_MASK = range(6)
F32, BF16, F64 = 0, 1, 2
SILU, GELU_ERF = 0, 1


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code


def build(force: bool = False) -> None:
    """Compile the restatement (and oracle/_ref when the reference is mounted)."""
    if force or not os.path.exists(_LIB_PATH):
        subprocess.check_call(["make", "-s", "liblkv_oracle.so"], cwd=_HERE)
    if os.path.isdir("/root/reference/proj/src"):
        subprocess.check_call(["make", "-s", "ref"], cwd=_HERE)


_lib = None
_ref = None

_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_ip = C.POINTER(C.c_int32)
_lp = C.POINTER(C.c_int64)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        L.lkvo_last_error.restype = C.c_char_p
        L.lkvo_laplace_cdf.restype = C.c_double
        L.lkvo_laplace_cdf.argtypes = [C.c_double]
        L.lkvo_bisect_lambda.restype = C.c_double
        L.lkvo_bisect_lambda.argtypes = [_dp, C.c_int, C.c_double, C.c_double]
        L.lkvo_solve_threshold.argtypes = [_dp, C.c_int, C.c_double, _dp, C.POINTER(C.c_int)]
        L.lkvo_soft_topk_forward.argtypes = [_dp, C.c_int, C.c_double, C.c_double, _dp, _dp,
                                             C.POINTER(C.c_int), _dp]
        L.lkvo_hard_topk.argtypes = [_dp, C.c_int, C.c_int, _ip]
        L.lkvo_select_positions_f32.argtypes = [_fp, C.c_int, C.c_int, _ip]
        L.lkvo_allocate_budgets.argtypes = [_dp, C.c_int, C.c_double, _dp]
        L.lkvo_freeze_budgets.argtypes = [_dp, C.c_int, C.c_int, _ip]
        L.lkvo_freeze_budgets_exact.argtypes = [_dp, C.c_int, C.c_double, C.c_int, _ip]
        L.lkvo_token_scores.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int,
                                        _dp, _dp, _dp, C.c_int, C.c_int, _dp]
        L.lkvo_compact_rows.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_int, _ip, C.c_int,
                                        C.c_void_p, C.c_void_p]
        L.lkvo_compact_rows.restype = None
        L.lkvo_decode_attention.argtypes = [C.c_int, _dp, C.c_int, C.c_void_p, C.c_void_p, C.c_int64,
                                            C.c_int, C.c_double, _dp]
        L.lkvo_soft_topk_density.argtypes = [_dp, C.c_int, C.c_double, C.c_double, C.c_double, _dp]
        L.lkvo_soft_topk_vjp.argtypes = [_dp, _dp, C.c_int, C.c_double, _dp, _dp]
        L.lkvo_masked_attention.argtypes = [_dp, _dp, _dp, _dp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                            C.c_int, C.c_int, _dp, _dp, _dp, _dp]
        L.lkvo_masked_attention_vjp.argtypes = [_dp, _dp, _dp, _dp, C.c_int, C.c_int, C.c_int, C.c_int,
                                                C.c_double, C.c_int, C.c_int, _dp, _dp, _dp, _dp, _dp]
        L.lkvo_kv_memory_bytes.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_int64, C.c_double,
                                           _dp, _dp, _dp]
        L.lkvo_kv_memory_bytes_budgets.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_int64,
                                                   _ip, C.c_int, _dp, _dp, _dp]
        L.lkvo_evict_heads.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int64, _ip, C.c_int,
                                       C.c_int, _dp, _dp, _dp, C.c_int, C.c_int, _ip, _ip, _lp,
                                       C.c_void_p, C.c_void_p, _ip, _dp, C.c_int]
        L.lkvo_rng_next.restype = C.c_uint64
        L.lkvo_rng_uniform.restype = C.c_double
        L.lkvo_rng_uniform_range.restype = C.c_double
        L.lkvo_rng_uniform_range.argtypes = [C.c_void_p, C.c_double, C.c_double]
        L.lkvo_rng_uniform_int.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.lkvo_rng_normal.restype = C.c_double
        L.lkvo_rng_seed.argtypes = [C.c_void_p, C.c_uint64]
        L.lkvo_rng_seed.restype = None
        L.lkvo_fill_uniform.argtypes = [C.c_uint64, C.c_double, C.c_double, _dp, C.c_int64]
        L.lkvo_fill_uniform.restype = None
        L.lkvo_mix64.restype = C.c_uint64
        L.lkvo_mix64.argtypes = [C.c_uint64]
        L.lkvo_derive_seed.restype = C.c_uint64
        L.lkvo_derive_seed.argtypes = [C.c_uint64] * 4
        _lib = L
    return _lib


def ref_lib():
    """The reference's own soft_topk.cpp/policy.cpp (None when not built here)."""
    global _ref
    if _ref is None and os.path.exists(_REF_PATH):
        R = C.CDLL(_REF_PATH)
        R.ref_solve_threshold.argtypes = [_dp, C.c_int, C.c_double, _dp, C.POINTER(C.c_int)]
        R.ref_soft_topk_forward.argtypes = [_dp, C.c_int, C.c_double, C.c_double, _dp, _dp,
                                            C.POINTER(C.c_int)]
        R.ref_allocate_budgets.argtypes = [_dp, C.c_int, C.c_int, C.c_double, _dp]
        R.ref_freeze_budgets.argtypes = [_dp, C.c_int, C.c_int, C.c_int, _ip]
        R.ref_hard_topk.argtypes = [_dp, C.c_int, C.c_int, _ip]
        R.ref_token_scores.argtypes = [_dp, _dp, C.c_int, C.c_int, _dp, _dp, _dp, C.c_int, _dp]
        R.ref_soft_topk_vjp.argtypes = [_dp, C.c_int, C.c_double, C.c_double, _dp, _dp, _dp, _dp, _dp]
        R.ref_masked_attention.argtypes = [_dp, _dp, _dp, _dp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                           C.c_int, C.c_int, _dp, _dp, _dp, _dp, _dp, _dp]
        _ref = R
    return _ref


def _check(rc: int) -> None:
    if rc != OK:
        raise OracleError(rc, lib().lkvo_last_error().decode())


def _d(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a, t):
    return a.ctypes.data_as(t)


# ---- reference rng (rng.hpp) --------------------------------------------------
class Rng:
    """lkv::Rng (rng.hpp:29-66): mt19937_64 with the reference's conversions."""

    def __init__(self, seed: int):
        self._state = C.create_string_buffer(312 * 8 + 64)
        lib().lkvo_rng_seed(self._state, C.c_uint64(seed & (2**64 - 1)))

    def next_u64(self) -> int:
        return lib().lkvo_rng_next(self._state)

    def uniform(self, lo: float = 0.0, hi: float = 1.0) -> float:
        return lib().lkvo_rng_uniform_range(self._state, lo, hi)

    def uniform_int(self, lo: int, hi: int) -> int:
        return lib().lkvo_rng_uniform_int(self._state, lo, hi)

    def normal(self) -> float:
        return lib().lkvo_rng_normal(self._state)


def mix64(z: int) -> int:
    return lib().lkvo_mix64(z & (2**64 - 1))


def derive_seed(base: int, a: int, b: int = 0, c: int = 0) -> int:
    return lib().lkvo_derive_seed(base, a, b, c)


def random_scores(n: int, seed: int, lo: float = -3.0, hi: float = 3.0) -> np.ndarray:
    """test_soft_topk.cpp:17-22."""
    out = np.empty(n, np.float64)
    lib().lkvo_fill_uniform(seed, lo, hi, _ptr(out, _dp), n)
    return out


# ---- soft_topk.cpp --------------------------------------------------------------
def laplace_cdf(z: float) -> float:
    return lib().lkvo_laplace_cdf(z)


def solve_threshold(x, k: float):
    x = _d(x)
    lam = C.c_double()
    m = C.c_int()
    _check(lib().lkvo_solve_threshold(_ptr(x, _dp), len(x), k, C.byref(lam), C.byref(m)))
    return lam.value, m.value


def soft_topk_forward(x, k: float, tau: float):
    x = _d(x)
    vals = np.empty(len(x), np.float64)
    lam = C.c_double()
    m = C.c_int()
    kc = C.c_double()
    _check(lib().lkvo_soft_topk_forward(_ptr(x, _dp), len(x), k, tau, _ptr(vals, _dp), C.byref(lam),
                                        C.byref(m), C.byref(kc)))
    return {"values": vals, "threshold_lambda": lam.value, "split_m": m.value, "clamped_k": kc.value}


def bisect_lambda(x, k: float, tol: float = 1e-12) -> float:
    x = _d(x)
    return lib().lkvo_bisect_lambda(_ptr(x, _dp), len(x), k, tol)


def hard_topk(x, b: int) -> np.ndarray:
    x = _d(x)
    mask = np.zeros(len(x), np.int32)
    _check(lib().lkvo_hard_topk(_ptr(x, _dp), len(x), b, _ptr(mask, _ip)))
    return mask


def select_positions_f32(x, b: int) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32)
    pos = np.zeros(max(b, 1), np.int32)
    _check(lib().lkvo_select_positions_f32(_ptr(x, _fp), len(x), b, _ptr(pos, _ip)))
    return pos[:b]


# ---- policy.cpp -----------------------------------------------------------------
def allocate_budgets(logits, target_ratio: float) -> np.ndarray:
    x = _d(logits)
    r = np.empty(len(x), np.float64)
    _check(lib().lkvo_allocate_budgets(_ptr(x, _dp), len(x), target_ratio, _ptr(r, _dp)))
    return r


def freeze_budgets(ratios, t: int) -> np.ndarray:
    r = _d(ratios)
    b = np.empty(len(r), np.int32)
    _check(lib().lkvo_freeze_budgets(_ptr(r, _dp), len(r), t, _ptr(b, _ip)))
    return b


def freeze_budgets_exact(ratios, target_ratio: float, t: int) -> np.ndarray:
    r = _d(ratios)
    b = np.empty(len(r), np.int32)
    _check(lib().lkvo_freeze_budgets_exact(_ptr(r, _dp), len(r), target_ratio, t, _ptr(b, _ip)))
    return b


def token_scores(keys, values, w1, b1, w2, act: int = SILU, dtype: int | None = None) -> np.ndarray:
    """keys/values: numpy [t][d] float32, float64 (widened) or uint16 (bf16 bits).
    values=None selects the K-only (in = d) scorer."""
    keys = np.ascontiguousarray(keys)
    if dtype is None:
        if keys.dtype == np.uint16:
            dtype = BF16
        else:
            dtype = F32
    if dtype == F32:
        keys = np.ascontiguousarray(keys, dtype=np.float32)
    elif dtype == F64:
        keys = np.ascontiguousarray(keys, dtype=np.float64)
    t, d = keys.shape
    in_mode = 1
    vptr = None
    if values is not None:
        values = np.ascontiguousarray(values, dtype=keys.dtype)
        in_mode = 2
        vptr = values.ctypes.data
    w1, b1, w2 = _d(w1), _d(b1), _d(w2).reshape(-1)
    hidden = w1.shape[1]
    assert w1.shape[0] == in_mode * d
    out = np.empty(t, np.float64)
    _check(lib().lkvo_token_scores(dtype, keys.ctypes.data, vptr, t, d, in_mode, _ptr(w1, _dp), _ptr(b1, _dp),
                                   _ptr(w2, _dp), hidden, act, _ptr(out, _dp)))
    return out


# ---- decode attention / memory model ----------------------------------------------
def decode_attention(q, keys, values, scale: float) -> np.ndarray:
    """q [G][d] fp64; keys/values [t][d] (float32 or uint16 bf16 bits)."""
    q = _d(q)
    keys = np.ascontiguousarray(keys)
    values = np.ascontiguousarray(values)
    dtype = BF16 if keys.dtype == np.uint16 else F32
    if dtype == F32:
        keys = np.ascontiguousarray(keys, np.float32)
        values = np.ascontiguousarray(values, np.float32)
    G, d = q.shape
    out = np.empty((G, d), np.float64)
    _check(lib().lkvo_decode_attention(dtype, _ptr(q, _dp), G, keys.ctypes.data, values.ctypes.data,
                                       keys.shape[0], d, scale, _ptr(out, _dp)))
    return out


# ---- training-time operators ---------------------------------
def soft_topk_full(x, k: float, tau: float = 1.0):
    """soft_topk_forward (soft_topk.cpp:111-164) -> (values, lambda, clamped_k, density_terms)."""
    x = _d(x)
    n = x.size
    vals = np.empty(n, np.float64)
    lam, m, kc = C.c_double(), C.c_int(), C.c_double()
    _check(lib().lkvo_soft_topk_forward(_ptr(x, _dp), n, k, tau, _ptr(vals, _dp), C.byref(lam), C.byref(m),
                                        C.byref(kc)))
    dens = np.empty(n, np.float64)
    _check(lib().lkvo_soft_topk_density(_ptr(x, _dp), n, tau, lam.value, kc.value, _ptr(dens, _dp)))
    return vals, lam.value, kc.value, dens


def soft_topk_vjp(density, upstream, tau: float = 1.0):
    """soft_topk_vjp (soft_topk.cpp:166-189) -> (grad_x, grad_k)."""
    density, upstream = _d(density), _d(upstream)
    gx = np.empty(density.size, np.float64)
    gk = C.c_double()
    _check(lib().lkvo_soft_topk_vjp(_ptr(density, _dp), _ptr(upstream, _dp), density.size, tau, _ptr(gx, _dp),
                                    C.byref(gk)))
    return gx, gk.value


def masked_attention(q, k, v, mask=None, causal=True, scale=None, pos_offset=0, self_keep=False, upstream=None):
    """masked_attention_dense (+ masked_attention_vjp when `upstream` is given), one head, fp64:
    q [n_q][d], k/v [t][d], mask [t] or None.  Returns out, or (out, dq, dk, dv, dmask)."""
    q, k, v = _d(q), _d(k), _d(v)
    n_q, d = q.shape
    t = k.shape[0]
    scale = 1.0 / np.sqrt(d) if scale is None else scale
    m = _d(mask) if mask is not None else None
    mp = _ptr(m, _dp) if m is not None else None
    out = np.empty((n_q, d), np.float64)
    _check(lib().lkvo_masked_attention(_ptr(q, _dp), _ptr(k, _dp), _ptr(v, _dp), mp, n_q, t, d, int(causal), scale,
                                       pos_offset, int(self_keep), _ptr(out, _dp), None, None, None))
    if upstream is None:
        return out
    u = _d(upstream)
    dq, dk, dv = np.zeros_like(q), np.zeros_like(k), np.zeros_like(v)
    dm = np.zeros(t, np.float64) if m is not None else None
    _check(lib().lkvo_masked_attention_vjp(_ptr(q, _dp), _ptr(k, _dp), _ptr(v, _dp), mp, n_q, t, d, int(causal),
                                           scale, pos_offset, int(self_keep), _ptr(u, _dp), _ptr(dq, _dp),
                                           _ptr(dk, _dp), _ptr(dv, _dp), _ptr(dm, _dp) if dm is not None else None))
    return out, dq, dk, dv, dm


def kv_memory_bytes(n_layers=32, n_kv_heads=8, head_dim=128, bytes_per_element=2.0, tokens=200000,
                    retention=None, budgets=None):
    full, comp, red = C.c_double(), C.c_double(), C.c_double()
    if budgets is not None:
        b = np.ascontiguousarray(budgets, np.int32)
        _check(lib().lkvo_kv_memory_bytes_budgets(n_layers, n_kv_heads, head_dim, bytes_per_element, tokens,
                                                  _ptr(b, _ip), len(b), C.byref(full), C.byref(comp),
                                                  C.byref(red)))
    else:
        _check(lib().lkvo_kv_memory_bytes(n_layers, n_kv_heads, head_dim, bytes_per_element, tokens,
                                          retention, C.byref(full), C.byref(comp), C.byref(red)))
    return {"full_bytes": full.value, "compressed_bytes": comp.value, "reduction_factor": red.value}


_fast = None


def fast_lib():
    """liblkv_oracle_fast.so (timing of the CPU baseline only; never a parity reference)."""
    global _fast
    if _fast is None:
        if not os.path.exists(_FAST_PATH):
            subprocess.check_call(["make", "-s", "liblkv_oracle_fast.so"], cwd=_HERE)
        L = C.CDLL(_FAST_PATH)
        L.lkvo_last_error.restype = C.c_char_p
        L.lkvo_evict_heads.argtypes = lib().lkvo_evict_heads.argtypes
        for name in ("lkvo_allocate_budgets", "lkvo_freeze_budgets_exact"):
            getattr(L, name).argtypes = getattr(lib(), name).argtypes
        _fast = L
    return _fast


def evict_heads(keys, values, t_per_head, in_mode, w1_all, b1_all, w2_all, act, head_scorer, budgets,
                offsets, n_threads=1, want_scores=False, fast=False):
    """Whole CPU eviction over heads.  keys/values: numpy [n_heads][T][d] (float32 or
    uint16 bf16 bits).  Returns (dst_k, dst_v, dst_pos[, scores])."""
    keys = np.ascontiguousarray(keys)
    values = np.ascontiguousarray(values)
    dtype = BF16 if keys.dtype == np.uint16 else F32
    n_heads, T, d = keys.shape
    w1_all, b1_all, w2_all = _d(w1_all), _d(b1_all), _d(w2_all)
    hidden = b1_all.shape[-1]
    t_per_head = np.ascontiguousarray(t_per_head, np.int32)
    head_scorer = np.ascontiguousarray(head_scorer, np.int32)
    budgets = np.ascontiguousarray(budgets, np.int32)
    offsets = np.ascontiguousarray(offsets, np.int64)
    total = int(offsets[-1])
    dst_k = np.zeros((max(total, 1), d), keys.dtype)
    dst_v = np.zeros((max(total, 1), d), keys.dtype)
    dst_pos = np.full(max(total, 1), -1, np.int32)
    scores = np.zeros((n_heads, T), np.float64) if want_scores else None
    L = fast_lib() if fast else lib()
    _check(L.lkvo_evict_heads(dtype, keys.ctypes.data, values.ctypes.data, n_heads, T,
                                  _ptr(t_per_head, _ip), d, in_mode, _ptr(w1_all, _dp), _ptr(b1_all, _dp),
                                  _ptr(w2_all, _dp), hidden, act, _ptr(head_scorer, _ip), _ptr(budgets, _ip),
                                  _ptr(offsets, _lp), dst_k.ctypes.data, dst_v.ctypes.data, _ptr(dst_pos, _ip),
                                  _ptr(scores, _dp) if want_scores else None, n_threads))
    if want_scores:
        return dst_k, dst_v, dst_pos, scores
    return dst_k, dst_v, dst_pos


# ---- bf16 helpers (host side of the same rounding the device sees) ---------------
def f32_to_bf16_bits(x) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 bit pattern (what torch .to(bfloat16) does)."""
    x = np.ascontiguousarray(x, np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    rounding = ((u >> 16) & 1) + 0x7FFF
    out = ((u + rounding) >> 16).astype(np.uint16)
    nan = np.isnan(x)
    if nan.any():
        out[nan] = 0x7FC0
    return out


def bf16_bits_to_f64(b) -> np.ndarray:
    b = np.ascontiguousarray(b, np.uint16)
    return (b.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
