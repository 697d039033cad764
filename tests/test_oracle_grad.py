"""Pins of the oracle gradient (O13: d ell / d theta for
theta = (sigma2, beta, tau2), nu fixed) to things other than itself:

* central finite differences of the oracle log-likelihood (itself pinned to
  dense Eq.1, tests/test_oracle_pins.py), per block and in total;
* full conditioning: the block-Vecchia gradient equals the gradient of the
  dense Eq.1 likelihood, computed with numpy as 1/2 tr((a a^T - K^-1) dK)
  where dK comes from central differences of the independent numpy
  covariance of tests/test_oracle_pins.dense_cov (scipy Bessel K_nu);
* the per-entry kernel derivative against central differences of the
  scipy-Bessel Matern.
"""
import numpy as np
import pytest

import sbv_inputs as si
from tests.test_oracle_pins import dense_cov, dense_loglik


def _fd(f, theta, k, rel=1e-5):
    h = rel * theta[k]
    tp, tm = theta.copy(), theta.copy()
    tp[k] += h
    tm[k] -= h
    return (f(tp) - f(tm)) / (2 * h)


def _grad_index(d):
    # theta = {sigma2, beta_1..beta_d, nu, tau2}; gradient order (sigma2, beta.., tau2)
    return [0] + list(range(1, d + 1)) + [d + 2]


@pytest.mark.parametrize("nu", [0.5, 1.5, 2.5, 3.5])
def test_kernel_derivative_matches_bessel_fd(orc, nu):
    rng = np.random.default_rng(5)
    d = 3
    theta = np.array([1.3, 0.4, 0.7, 1.1, nu, 1e-3])
    for _ in range(20):
        xa, xb = rng.random(d), rng.random(d)
        g = orc.kernel_grad(xa, xb, theta, False)
        for gi, k in enumerate(_grad_index(d)):
            f = lambda th: dense_cov(np.stack([xa, xb]), th)[0, 1]
            ref = _fd(f, theta, k)
            assert abs(g[gi] - ref) <= 1e-7 * max(1e-3, abs(ref)), (nu, k, g[gi], ref)
    # same point: d/dsigma2 = 1, d/dbeta = 0, d/dtau2 = 1
    g = orc.kernel_grad(xa, xa, theta, True)
    assert g[0] == 1.0 and np.all(g[1:1 + d] == 0.0) and g[-1] == 1.0


@pytest.mark.parametrize("nu", [1.5, 2.5, 3.5])
def test_block_gradient_matches_finite_differences(orc, nu):
    n, d, bs, m = 240, 3, 12, 20
    X = si.make_X(n, d, seed=61)
    y = si.make_y(X, seed=62)
    theta = np.array([1.2, 0.3, 0.5, 0.9, nu, 1e-2])
    P = orc.prepare(X, bs, m, theta[1:1 + d], 3)
    g, gb = orc.loglik_grad(X, y, P["perm"], P["off"], P["nbr"], P["cnt"], theta, return_blocks=True)
    ll = lambda th: orc.loglik(X, y, P["perm"], P["off"], P["nbr"], P["cnt"], th)
    for gi, k in enumerate(_grad_index(d)):
        ref = _fd(ll, theta, k)
        assert abs(g[gi] - ref) <= 2e-6 * max(1.0, abs(ref)), (k, g[gi], ref)
    # one block on its own
    t = 7
    J, B = P["nbr"][t, :P["cnt"][t]], P["perm"][P["off"][t]:P["off"][t + 1]]
    bt = lambda th: orc.block_term(X, y, J, B, th)[0]
    gt = orc.block_grad(X, y, J, B, theta)
    np.testing.assert_array_equal(gt, gb[t])
    for gi, k in enumerate(_grad_index(d)):
        ref = _fd(bt, theta, k)
        assert abs(gt[gi] - ref) <= 2e-6 * max(1.0, abs(ref)), (k, gt[gi], ref)


@pytest.mark.parametrize("bs", [1, 10])
def test_full_conditioning_gradient_equals_dense(orc, bs):
    """m >= n: sum_t d ell_t = d ell_dense (Eq.1), the dense gradient by numpy."""
    n, d = 90, 3
    X = si.make_X(n, d, seed=71)
    y = si.make_y(X, seed=72)
    theta = np.array([1.1, 0.5, 0.8, 0.6, 2.5, 1e-2])
    P = orc.prepare(X, bs, n - 1, theta[1:1 + d], 3)
    g = orc.loglik_grad(X, y, P["perm"], P["off"], P["nbr"], P["cnt"], theta)
    K = dense_cov(X, theta)
    Kinv = np.linalg.inv(K)
    a = Kinv @ y
    for gi, k in enumerate(_grad_index(d)):
        dK = _fd(lambda th: dense_cov(X, th), theta, k, rel=1e-6)
        ref = 0.5 * (a @ dK @ a - np.trace(Kinv @ dK))
        assert abs(g[gi] - ref) <= 1e-6 * max(1.0, abs(ref)), (k, g[gi], ref)
    # and against finite differences of the dense Eq.1 log-likelihood itself
    for gi, k in enumerate(_grad_index(d)):
        ref = _fd(lambda th: dense_loglik(X, y, th), theta, k)
        assert abs(g[gi] - ref) <= 1e-5 * max(1.0, abs(ref)), (k, g[gi], ref)


def test_gradient_rejects_general_nu(orc):
    X = si.make_X(30, 2, seed=1)
    y = si.make_y(X, seed=2)
    with pytest.raises(ValueError):
        orc.block_grad(X, y, [0, 1], [2, 3], np.array([1.0, 0.5, 0.5, 1.3, 1e-3]))
