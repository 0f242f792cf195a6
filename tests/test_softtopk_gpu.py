"""GPU Soft-TopK forward / VJP against the oracle's restatement of
soft_topk_forward / soft_topk_vjp (pinned bit-exact to the reference on CPU,
tests/test_oracle_train.py).  fp64 throughout: values and gradients within 1e-10 absolute,
lambda within 1e-10 relative (only the summation order differs from the reference)."""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2605_06676_b200 as lkv
from paper_2605_06676_b200 import train

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n_seg,n,tau,sigma", [(8, 256, 1.0, 1.0), (3, 5000, 0.7, 2.0), (2, 40000, 1.3, 1.0),
                                               (16, 3, 1.0, 0.5), (4, 1, 1.0, 1.0), (5, 640, 1.0, 1.5)])
def test_soft_topk_matches_oracle(n_seg, n, tau, sigma):
    rng = np.random.default_rng(n_seg * 1000 + n)
    x = rng.normal(0, sigma, (n_seg, n))
    if n > 10:
        x[0, : n // 4] = np.round(x[0, : n // 4], 1)  # ties
    k = rng.uniform(0.05, 0.95, n_seg) * n
    if n == 1:
        k = rng.uniform(0.05, 0.95, n_seg)
    u = rng.normal(size=(n_seg, n))
    xt = torch.tensor(x, device="cuda")
    vals, dens, lam, v32 = train.soft_topk(xt, torch.tensor(k, device="cuda"), tau, f32_mask=True)
    gx, gk = train.soft_topk_vjp(dens, torch.tensor(u, device="cuda"), tau)
    for s in range(n_seg):
        rv, rlam, rkc, rd = O.soft_topk_full(x[s], k[s], tau)
        rgx, rgk = O.soft_topk_vjp(rd, u[s], tau)
        assert np.max(np.abs(vals[s].cpu().numpy() - rv)) <= 1e-10
        assert np.max(np.abs(dens[s].cpu().numpy() - rd)) <= 1e-10
        assert abs(float(lam[s]) - rlam) <= 1e-10 * max(1.0, abs(rlam))
        assert np.max(np.abs(gx[s].cpu().numpy() - rgx)) <= 1e-10
        assert abs(float(gk[s]) - rgk) <= 1e-10 * max(1.0, abs(rgk))
        assert np.max(np.abs(v32[s].cpu().numpy() - rv.astype(np.float32))) == 0.0
        assert abs(float(vals[s].sum()) - rkc) <= 1e-9 * n  # the reference's constraint check


def test_soft_topk_unit_upstream_is_exact():
    """test_soft_topk.cpp:129-136 on the device: unit upstream -> grad_x == 0, grad_k == 1."""
    x = torch.randn(6, 3001, dtype=torch.float64, device="cuda")
    _, dens, _, _ = train.soft_topk(x, torch.full((6,), 700.3, dtype=torch.float64, device="cuda"), 0.7)
    gx, gk = train.soft_topk_vjp(dens, torch.ones_like(x), 0.7)
    assert bool((gx == 0).all()) and bool((gk == 1).all())


def test_training_mask_with_noise_matches_oracle():
    """training_mask (policy.cpp:138-150): the soft top-k of u + noise_scale * gumbel."""
    rng = np.random.default_rng(3)
    u = rng.normal(size=(4, 2048))
    g = -np.log(-np.log(np.clip(rng.uniform(size=(4, 2048)), 1e-12, 1 - 1e-12)))
    vals, _, _, _ = train.soft_topk(torch.tensor(u, device="cuda"), 300.5, 0.5, noise=torch.tensor(g, device="cuda"),
                                    noise_scale=0.3)
    for s in range(4):
        rv, _, _, _ = O.soft_topk_full(u[s] + 0.3 * g[s], 300.5, 0.5)
        assert np.max(np.abs(vals[s].cpu().numpy() - rv)) <= 1e-10


def test_soft_topk_errors():
    x = torch.randn(2, 10, dtype=torch.float64, device="cuda")
    with pytest.raises(lkv.BudgetError):  # clamp_budget: k outside (0, n)
        train.soft_topk(x, torch.tensor([3.0, 10.0], dtype=torch.float64, device="cuda"))
    bad = x.clone()
    bad[1, 3] = float("nan")
    with pytest.raises(lkv.NumericError):
        train.soft_topk(bad, 3.0)
    big = x.clone()
    big[0, 0] = 1e301
    with pytest.raises(lkv.OverflowGuardError):
        train.soft_topk(big, 3.0)
    with pytest.raises(lkv.ContractError):
        train.soft_topk(x, 3.0, tau=0.0)
