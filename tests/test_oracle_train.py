"""CPU: the oracle's restatement of the training-time operators pinned against
the reference's own attention.cpp / soft_topk.cpp (oracle/_ref, compiled in place from
/root/reference) and against finite differences (the reference's gradcheck.cpp protocol)."""
import ctypes as C

import numpy as np
import pytest

import oracle as O

_dp = C.POINTER(C.c_double)


def _p(a):
    return a.ctypes.data_as(_dp) if a is not None else None


def _ref_attention(q, k, v, mask, causal, scale, off, self_keep, u):
    R = O.ref_lib()
    n_q, d = q.shape
    t = k.shape[0]
    out = np.empty((n_q, d))
    dq, dk, dv = np.empty((n_q, d)), np.empty((t, d)), np.empty((t, d))
    dm = np.empty(t) if mask is not None else None
    rc = R.ref_masked_attention(_p(q), _p(k), _p(v), _p(mask), n_q, t, d, int(causal), scale, off, int(self_keep),
                                _p(u), _p(out), _p(dq), _p(dk), _p(dv), _p(dm))
    return rc, (out, dq, dk, dv, dm)


needs_ref = pytest.mark.skipif(O.ref_lib() is None, reason="oracle/_ref not built (reference not mounted)")


@needs_ref
def test_masked_attention_oracle_equals_reference():
    rng = np.random.default_rng(11)
    for rep in range(40):
        n_q, t, d = int(rng.integers(1, 9)), int(rng.integers(1, 17)), int(rng.integers(1, 9))
        causal = bool(rng.integers(0, 2))
        off = int(rng.integers(0, max(1, t - n_q + 1))) if causal else 0
        self_keep = bool(rng.integers(0, 2))
        q, k, v, u = (rng.normal(size=s) for s in ((n_q, d), (t, d), (t, d), (n_q, d)))
        mask = rng.uniform(0, 1, t) if rep % 3 else None
        if mask is not None:
            mask[rng.uniform(size=t) < 0.3] = 0.0
            mask[0] = 0.5
        scale = float(rng.uniform(0.1, 1.0))
        rc, ref = _ref_attention(q, k, v, mask, causal, scale, off, self_keep, u)
        if rc != 0:
            with pytest.raises(O.OracleError):
                O.masked_attention(q, k, v, mask, causal, scale, off, self_keep, upstream=u)
            continue
        got = O.masked_attention(q, k, v, mask, causal, scale, off, self_keep, upstream=u)
        for g, r in zip(got, ref):
            if r is None:
                assert g is None
            else:
                assert np.array_equal(g, r)  # same operation order -> bit-identical


@needs_ref
def test_soft_topk_vjp_oracle_equals_reference():
    R = O.ref_lib()
    rng = np.random.default_rng(5)
    for rep in range(40):
        n = int(rng.integers(1, 300))
        x = rng.normal(0, 2, n)
        k = float(rng.uniform(0.05, 0.95)) * n if n > 1 else 0.4
        tau = float(rng.uniform(0.3, 2.0))
        u = rng.normal(size=n)
        vals, dens, gx, gk = np.empty(n), np.empty(n), np.empty(n), C.c_double()
        rc = R.ref_soft_topk_vjp(_p(x), n, k, tau, _p(u), _p(vals), _p(dens), _p(gx), C.byref(gk))
        assert rc == 0
        v2, lam, kc, d2 = O.soft_topk_full(x, k, tau)
        g2, k2 = O.soft_topk_vjp(d2, u, tau)
        assert np.array_equal(v2, vals) and np.array_equal(d2, dens)
        assert np.array_equal(g2, gx) and k2 == gk.value


def test_soft_topk_vjp_known_answers():
    """test_soft_topk.cpp:129-136: a unit upstream gives an exactly zero score gradient and an
    exactly unit budget gradient; gradients match central differences (:138-170)."""
    rng = np.random.default_rng(2)
    x = rng.normal(size=40)
    _, _, _, dens = O.soft_topk_full(x, 12.5, 0.7)
    gx, gk = O.soft_topk_vjp(dens, np.ones(40), 0.7)
    assert np.all(gx == 0.0) and gk == 1.0
    u = rng.normal(size=40)
    gx, gk = O.soft_topk_vjp(dens, u, 0.7)
    h = 1e-6
    for i in (0, 7, 19):
        xp, xm = x.copy(), x.copy()
        xp[i] += h
        xm[i] -= h
        fd = (u @ O.soft_topk_full(xp, 12.5, 0.7)[0] - u @ O.soft_topk_full(xm, 12.5, 0.7)[0]) / (2 * h)
        assert abs(fd - gx[i]) <= 1e-6 * max(1.0, abs(fd))
    fdk = (u @ O.soft_topk_full(x, 12.5 + h, 0.7)[0] - u @ O.soft_topk_full(x, 12.5 - h, 0.7)[0]) / (2 * h)
    assert abs(fdk - gk) <= 1e-6 * max(1.0, abs(fdk))


def test_masked_attention_oracle_finite_differences():
    """attention gradients vs central differences of <u, out> (gradcheck.cpp:30-180 protocol)."""
    rng = np.random.default_rng(4)
    n_q, t, d = 5, 9, 4
    q, k, v, u = (rng.normal(size=s) for s in ((n_q, d), (t, d), (t, d), (n_q, d)))
    mask = rng.uniform(0.2, 1.0, t)
    args = (True, 0.6, 4, True)
    out, dq, dk, dv, dm = O.masked_attention(q, k, v, mask, *args, upstream=u)
    f = lambda q_, k_, v_, m_: float(np.sum(u * O.masked_attention(q_, k_, v_, m_, *args)))
    h = 1e-6
    for name, arr, grad in (("q", q, dq), ("k", k, dk), ("v", v, dv), ("m", mask, dm)):
        for idx in [(0,) * arr.ndim, tuple(s - 1 for s in arr.shape)]:
            ap, am = arr.copy(), arr.copy()
            ap[idx] += h
            am[idx] -= h
            bind = {"q": (ap, k, v, mask), "k": (q, ap, v, mask), "v": (q, k, ap, mask), "m": (q, k, v, ap)}[name]
            bindm = {"q": (am, k, v, mask), "k": (q, am, v, mask), "v": (q, k, am, mask), "m": (q, k, v, am)}[name]
            fd = (f(*bind) - f(*bindm)) / (2 * h)
            assert abs(fd - grad[idx]) <= 1e-6 * max(1.0, abs(fd)), (name, idx, fd, grad[idx])


def test_masked_attention_oracle_log_space_equivalence():
    """test_attention.cpp:63-71: the probability-domain mask equals softmax(s + log m) V."""
    rng = np.random.default_rng(8)
    q, k, v = rng.normal(size=(3, 5)), rng.normal(size=(11, 5)), rng.normal(size=(11, 5))
    m = rng.uniform(0.05, 1.0, 11)
    out = O.masked_attention(q, k, v, m, False, 0.4)
    s = 0.4 * q @ k.T + np.log(m)[None, :]
    p = np.exp(s - s.max(axis=1, keepdims=True))
    p /= p.sum(axis=1, keepdims=True)
    assert np.max(np.abs(out - p @ v)) <= 1e-12
