"""GPU parity of the gradient (sbv_loglik_grad) against the
oracle's O13 (explicit inverses; pinned in tests/test_oracle_grad.py).

Bar (Q28b): each component within 1e-7 of max(|g_k|, sum_t |g_t,k|)
(the per-block gradients are sums of terms that cancel; the same guard as the
log-likelihood's Q18), and ell bitwise equal to sbv_loglik's.
"""
import json
import os

import numpy as np
import pytest

import sbv_inputs as si

pytestmark = pytest.mark.gpu
TOL_G = 1e-7
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def sbv():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2504_12004_b200 as p
    from paper_2504_12004_b200 import build
    build.build()
    return p


def _check(sbv, orc, X, y, bs, m, scale, theta, name):
    import torch
    h = sbv.prepare(torch.from_numpy(X).cuda(), bs, m, scale)
    yt = torch.from_numpy(y).cuda()
    ll, g = h.loglik_grad(yt, theta)
    assert ll == h.loglik(yt, theta)
    P = orc.prepare(X, bs, m, scale, 3)
    go, gb = orc.loglik_grad(X, y, P["perm"], P["off"], P["nbr"], P["cnt"], theta, return_blocks=True)
    base = np.maximum(np.abs(go), np.abs(gb).sum(0))
    rel = np.abs(g - go) / base
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "parity_report.jsonl"), "a") as f:
        f.write(json.dumps({"test": name, "max_rel_grad": float(rel.max()),
                            "max_rel_grad_strict": float((np.abs(g - go) / np.maximum(np.abs(go), 1e-300)).max())}) + "\n")
    assert rel.max() <= TOL_G, (rel, g, go)
    gbg = h.block_grads()  # per block, zeta order (sbv_block_grads)
    assert np.all(np.abs(gbg - gb) <= TOL_G * np.abs(gb).sum(0)), np.abs(gbg - gb).max(0)
    return h, g


@pytest.mark.parametrize("nw", ["4", "8"])
def test_grad_both_cta_shapes(sbv, orc, nw, monkeypatch):
    """k_grad's 4-warp (2 CTAs/SM) and 8-warp instantiations (grad_shape picks
    by blocks per CTA; SBV_GRAD_NW forces one) against the oracle, N up to
    ~420 (b > 128: several Z slices per warp)."""
    monkeypatch.setenv("SBV_GRAD_NW", nw)
    n, d, bs, m = 4000, 5, 150, 200
    X = si.make_X(n, d, seed=9)
    y = si.make_y(X, seed=10)
    scale = si.default_scale(d)
    theta = si.default_theta(d, nu=2.5, tau2=1e-3)
    _check(sbv, orc, X, y, bs, m, scale, theta, f"grad_nw{nw}")


@pytest.mark.parametrize("d,bs,m,nu", [
    (5, 20, 40, 2.5),
    (3, 10, 30, 3.5),
    (2, 7, 13, 0.5),
    (10, 20, 60, 1.5),   # cfg1 shape (reduced n)
    (4, 1, 5, 2.5),      # bs = 1
    (3, 30, 0, 2.5),     # m = 0: marginal blocks only
])
def test_grad_parity_small(sbv, orc, d, bs, m, nu):
    n = 2000
    X = si.make_X(n, d, seed=30 + d)
    y = si.make_y(X, seed=40 + d)
    scale = si.default_scale(d)
    theta = si.default_theta(d, nu=nu, tau2=1e-3)
    _check(sbv, orc, X, y, bs, m, scale, theta, f"grad_small_d{d}_bs{bs}_m{m}_nu{nu}")


def test_grad_large_blocks_and_batches(sbv, orc, monkeypatch):
    """N_t up to ~600 (several 32-row panels, ragged tails) and the factor
    copies split over many batches (SBV_GRAD_BATCH_GB tiny): same gradient."""
    n, d, bs, m = 3000, 4, 250, 300
    X = si.make_X(n, d, seed=5)
    y = si.make_y(X, seed=6)
    scale = np.array([0.2, 0.3, 1.0, 2.0])
    theta = np.array([1.3, 0.2, 0.3, 1.0, 2.0, 2.5, 1e-3])
    h, g = _check(sbv, orc, X, y, bs, m, scale, theta, "grad_large_blocks")
    assert h.stats()["max_N"] > 500
    monkeypatch.setenv("SBV_GRAD_BATCH_GB", "0.002")
    ll2, g2 = h.loglik_grad(y, theta)
    np.testing.assert_array_equal(g2, g)


def test_grad_rejects_general_nu(sbv):
    X = si.make_X(500, 3, seed=1)
    h = sbv.prepare(X, 10, 20, np.ones(3))
    with pytest.raises(sbv.SBVError) as e:
        h.loglik_grad(np.zeros(500), np.array([1.0, 1, 1, 1, 1.3, 1e-3]))
    assert e.value.code == 5


def test_grad_cfg2_full_size_central_differences(sbv):
    """BASELINE cfg2 at full size (n = 1M, d = 10, bs = 100, m = 200, nu = 2.5,
    the bench's launch configuration) where the oracle's explicit inverses
    are out of reach: every gradient component against a central difference
    of sbv_loglik itself (parity-pinned to the oracle at 1e-9), steps 1e-3 and
    2e-3 relative with Richardson extrapolation (truncation O(h^4), leaving
    the rounding noise of the deterministic ell, which falls as 1/h:
    profiles/r02/grad_fd_check_cfg2.jsonl, 1e-6 ... 1e-3).  Same bar as the oracle tests
    (Q28b: 1e-7 of max(|g_k|, sum_t |g_t,k|), the per-block gradients from
    sbv_block_grads)."""
    import torch
    c = si.CONFIGS["cfg2"]
    n, d, bs, m = c["n"], c["d"], c["bs"], c["m"]
    Xh = si.make_X(n, d, seed=1)
    X = torch.from_numpy(Xh).cuda()
    y = torch.from_numpy(si.make_y(Xh, seed=2)).cuda()  # smooth field + noise (the input recipe)
    theta = si.default_theta(d, nu=c["nu"], tau2=1e-4)
    h = sbv.Handle(seed=3)
    h.prepare(X, bs, m, si.default_scale(d))
    ll, g = h.loglik_grad(y, theta)
    assert ll == h.loglik(y, theta)
    idx = [0, *range(1, d + 1), d + 2]  # sigma2, beta_1..beta_d, tau2 (nu fixed)
    fd = np.zeros(len(idx))

    def central(i, rel_step):
        tp, tm = theta.copy(), theta.copy()
        tp[i] += rel_step * theta[i]
        tm[i] -= rel_step * theta[i]
        return (h.loglik(y, tp) - h.loglik(y, tm)) / (tp[i] - tm[i])

    for k, i in enumerate(idx):  # Richardson: (4 D(h) - D(2h)) / 3 cancels the h^2 term
        fd[k] = (4.0 * central(i, 1e-3) - central(i, 2e-3)) / 3.0
    gb = h.block_grads()  # per-block gradients: the Q28b base max(|g|, sum_t |g_t|)
    assert gb.shape == (h.num_blocks(), d + 2)
    base = np.maximum(np.abs(g), np.abs(gb).sum(0))
    assert np.all(np.abs(gb.sum(0) - g) <= 1e-12 * base)
    rel = np.abs(g - fd) / base
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "parity_report.jsonl"), "a") as f:
        f.write(json.dumps({"test": "grad_cfg2_central_differences", "max_rel": float(rel.max()),
                            "rel": rel.tolist(), "rel_to_abs_g": (np.abs(g - fd) / np.abs(g)).tolist()}) + "\n")
    assert rel.max() <= TOL_G, (rel, g, fd)


def test_block_grads_state_rules(sbv):
    """sbv_block_grads: SBV_ERR_STATE before any sbv_loglik_grad and after a
    re-prepare; after a gradient call its rows sum to the gradient."""
    import torch
    n, d, bs, m = 3000, 4, 30, 40
    X = torch.from_numpy(si.make_X(n, d, seed=21)).cuda()
    y = torch.from_numpy(si.make_y(si.make_X(n, d, seed=21), seed=22)).cuda()
    theta = si.default_theta(d, nu=1.5, tau2=1e-3)
    h = sbv.Handle(seed=3)
    h.prepare(X, bs, m, si.default_scale(d))
    with pytest.raises(sbv.SBVError) as e:
        h.block_grads()
    state = e.value.code
    assert state == 7  # SBV_ERR_STATE
    ll, g = h.loglik_grad(y, theta)
    gb = h.block_grads()
    assert np.all(np.abs(gb.sum(0) - g) <= 1e-12 * np.abs(gb).sum(0))
    h.prepare(X, bs, m, si.default_scale(d))
    with pytest.raises(sbv.SBVError) as e:
        h.block_grads()
    assert e.value.code == state
