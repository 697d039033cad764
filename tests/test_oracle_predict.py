"""Pins for the oracle's prediction path (Eq.3 P:198-201,
Sec.4.1, Sec.5.5).

Each check ties oracle.predict / knn_pred / simulate / z_crit to something
other than the oracle itself: dense GP conditioning written with numpy and
scipy Bessel functions, closed-form limits, exact lattice distances, scipy's
normal quantile and the law of large numbers."""
import math

import numpy as np
import pytest
from scipy import stats

import sbv_inputs as si
from tests.test_oracle_pins import dense_cov, matern_bessel, rand_theta


def dense_predict(X, y, Xs, theta):
    """Sec.4.1: mu* = S*^T S^-1 y, diag(S** - S*^T S^-1 S*), via numpy."""
    d = X.shape[1]
    beta = theta[1:1 + d]
    Z, Zs = X / beta, Xs / beta
    Ds = np.sqrt(((Z[:, None, :] - Zs[None, :, :]) ** 2).sum(-1))
    Kx = matern_bessel(Ds, theta[0], theta[d + 1])  # n x n*
    S = dense_cov(X, theta)
    mu = Kx.T @ np.linalg.solve(S, y)
    var = theta[0] + theta[d + 2] - np.einsum("ij,ij->j", Kx, np.linalg.solve(S, Kx))
    return mu, var


@pytest.mark.parametrize("nu", [1.5, 2.5, 3.5])
def test_full_conditioning_equals_dense_prediction(orc, nu):
    """m_pred >= n: every test block conditions on all training points."""
    rng = np.random.default_rng(11)
    n, d = 120, 3
    X = rng.uniform(size=(n, d))
    y = rng.normal(size=n)
    Xs = rng.uniform(size=(25, d))
    theta = rand_theta(d, nu, 1e-3, rng)
    mu, var, _ = orc.predict(X, y, Xs, 4, n, theta[1:1 + d], theta)
    mu_d, var_d = dense_predict(X, y, Xs, theta)
    np.testing.assert_allclose(mu, mu_d, rtol=1e-8, atol=1e-9)
    np.testing.assert_allclose(var, var_d, rtol=1e-8, atol=1e-10)


def test_interpolation_at_training_points(orc):
    """tau^2 = 0, test point = training point in NN: mean = its y, var = 0."""
    rng = np.random.default_rng(3)
    n, d = 60, 2
    X = rng.uniform(size=(n, d))
    y = rng.normal(size=n)
    theta = np.array([1.0, 0.4, 0.7, 1.5, 0.0])
    idx = np.array([5, 17, 42])
    mu, var, _ = orc.predict(X, y, X[idx], 1, 20, theta[1:3], theta)
    np.testing.assert_allclose(mu, y[idx], atol=1e-8)
    assert np.all(np.abs(var) < 1e-8)


def test_far_test_point_reverts_to_prior(orc):
    """r >> range: mean -> 0, var -> sigma^2 + tau^2."""
    rng = np.random.default_rng(4)
    X = rng.uniform(size=(50, 2))
    y = rng.normal(size=50)
    theta = np.array([1.7, 0.1, 0.1, 2.5, 0.01])
    Xs = np.array([[1e3, 1e3], [-5e2, 7e2]])
    mu, var, _ = orc.predict(X, y, Xs, 1, 10, theta[1:3], theta)
    np.testing.assert_allclose(mu, 0.0, atol=1e-12)
    np.testing.assert_allclose(var, 1.71, rtol=1e-12)


def test_variance_never_increases_with_more_training_points(orc):
    """Nested designs, full conditioning: var at held-out points is monotone."""
    rng = np.random.default_rng(5)
    X = rng.uniform(size=(80, 3))
    y = rng.normal(size=80)
    Xs = rng.uniform(size=(10, 3))
    theta = rand_theta(3, 2.5, 1e-3, rng)
    prev = None
    for n in (20, 40, 80):
        _, var, _ = orc.predict(X[:n], y[:n], Xs, 2, n, theta[1:4], theta)
        if prev is not None:
            assert np.all(var <= prev + 1e-12)
        prev = var


def test_knn_pred_exact_on_lattice(orc):
    """Prediction-mode NN = all training points by (d2, index), lattice data
    so squared distances are exact integers; ties go to the lower index."""
    g = np.arange(6, dtype=np.float64)
    S = np.array(np.meshgrid(g, g, g, indexing="ij")).reshape(3, -1).T.copy()  # 216 points
    rng = np.random.default_rng(6)
    for _ in range(20):
        c = rng.integers(0, 6, size=3).astype(np.float64) + rng.choice([0.0, 0.5], size=3)
        d2 = ((S - c) ** 2).sum(1)
        ref = np.lexsort((np.arange(S.shape[0]), d2))[:17]
        np.testing.assert_array_equal(orc.knn_pred(S, c, 17), ref)


def test_z_crit_matches_normal_quantile(orc):
    for ci in (0.8, 0.9, 0.95, 0.99):
        assert abs(orc.z_crit(ci) - stats.norm.ppf(0.5 + ci / 2)) < 1e-12


def test_simulation_law_of_large_numbers(orc):
    """n_sim -> inf: sample mean -> mean, sample sd -> sqrt(var), within 4 MC sigmas."""
    mean = np.array([0.3, -2.0, 5.0])
    var = np.array([1.0, 0.25, 4.0])
    n_sim = 100_000
    sm, ssd, lo, hi = orc.simulate(mean, var, n_sim, seed=9)
    sd = np.sqrt(var)
    assert np.all(np.abs(sm - mean) < 4 * sd / math.sqrt(n_sim))
    assert np.all(np.abs(ssd - sd) < 4 * sd / math.sqrt(2 * n_sim))
    z = stats.norm.ppf(0.975)
    np.testing.assert_allclose(lo, sm - z * ssd, rtol=1e-13)
    np.testing.assert_allclose(hi, sm + z * ssd, rtol=1e-13)


def test_simulation_zero_variance_is_degenerate(orc):
    sm, ssd, lo, hi = orc.simulate(np.array([1.25]), np.array([0.0]), 1000, seed=1)
    assert sm[0] == 1.25 and ssd[0] == 0.0 and lo[0] == 1.25 and hi[0] == 1.25
