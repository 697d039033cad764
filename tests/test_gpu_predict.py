"""GPU parity of the prediction path against the CPU oracle.

Bar: test anchors / blocks / layout and the prediction-mode conditioning sets
bit-exact; mean within 1e-9 * max(1, |y|_inf) and variance within
1e-9 * (sigma^2 + tau^2) absolute (Q25: the GPU reads both off the
joint factor, the oracle uses the explicit Sec.4.1 formulas); simulation
within 1e-12 relative of the oracle's (same counter-based draws, libm ulps)."""
import numpy as np
import pytest

import sbv_inputs as si

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sbv():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2504_12004_b200 as p
    from paper_2504_12004_b200 import build
    build.build()
    return p


def check(h, orc, X, y, Xs, bs_pred, m_pred, theta, scale, seed=3, device=False):
    import torch
    Xa = torch.from_numpy(Xs).cuda() if device else Xs
    ya = torch.from_numpy(y).cuda() if device else y
    mean, var = h.predict(Xa, bs_pred, m_pred, ya, theta)
    if device:
        mean, var = mean.cpu().numpy(), var.cpu().numpy()
    mo, vo, info = orc.predict(X, y, Xs, bs_pred, m_pred, scale, theta, seed)
    anc, bo, off, perm, nbr, cnt = h.prediction_structure()
    np.testing.assert_array_equal(anc, info["anchors"])
    np.testing.assert_array_equal(bo, info["block_of"])
    np.testing.assert_array_equal(off, info["off"])
    np.testing.assert_array_equal(perm, info["perm"])
    for t, J in enumerate(info["nbr"]):
        assert cnt[t] == len(J), t
        np.testing.assert_array_equal(nbr[t, :cnt[t]], J, err_msg=f"test block {t}")
    d = X.shape[1]
    tol_m = 1e-9 * max(1.0, np.abs(y).max())
    tol_v = 1e-9 * (theta[0] + theta[d + 2])
    assert np.abs(mean - mo).max() <= tol_m, np.abs(mean - mo).max()
    assert np.abs(var - vo).max() <= tol_v, np.abs(var - vo).max()
    return mean, var


@pytest.mark.parametrize("d,bs_pred,m_pred,nu", [
    (10, 10, 60, 2.5),
    (3, 1, 20, 1.5),     # bs_pred = 1: point-wise prediction
    (5, 40, 90, 3.5),
    (2, 7, 0, 0.5),      # m_pred = 0: prior variance
])
def test_predict_parity(sbv, orc, d, bs_pred, m_pred, nu):
    n, ns = 4000, 700
    X = si.make_X(n, d, seed=50 + d)
    y = si.make_y(X, seed=60 + d)
    Xs = si.make_X(ns, d, seed=70 + d)
    sc = si.default_scale(d)
    theta = si.default_theta(d, nu=nu, tau2=1e-4)
    h = sbv.prepare(X, 20, 40, sc)
    check(h, orc, X, y, Xs, bs_pred, m_pred, theta, sc)


def test_predict_device_inputs_and_interpolation(sbv, orc):
    """CUDA-tensor inputs; test points at training points with tau^2 = 0 and
    bs_pred = 1: mean = y, var = 0 on the GPU path."""
    n, d = 3000, 4
    X = si.make_X(n, d, seed=81)
    y = si.make_y(X, seed=82)
    theta = np.array([1.0, 0.3, 0.4, 0.5, 0.6, 2.5, 0.0])
    sc = theta[1:1 + d].copy()
    h = sbv.prepare(X, 10, 30, sc)
    idx = np.arange(0, n, 97)
    mean, var = check(h, orc, X, y, X[idx], 1, 25, theta, sc, device=True)
    np.testing.assert_allclose(mean, y[idx], atol=1e-8)
    assert np.abs(var).max() < 1e-8


def test_predict_full_conditioning_equals_dense(sbv):
    """m_pred >= n: the GPU prediction is the exact GP prediction (Sec.4.1)."""
    from tests.test_oracle_predict import dense_predict
    rng = np.random.default_rng(9)
    n, d = 300, 3
    X = rng.uniform(size=(n, d))
    y = rng.normal(size=n)
    Xs = rng.uniform(size=(60, d))
    theta = np.array([1.2, 0.5, 0.8, 1.1, 2.5, 1e-3])
    h = sbv.prepare(X, 10, 50, theta[1:1 + d])
    mean, var = h.predict(Xs, 6, n, y, theta)
    mu_d, var_d = dense_predict(X, y, Xs, theta)
    np.testing.assert_allclose(mean, mu_d, rtol=1e-8, atol=1e-9)
    np.testing.assert_allclose(var, var_d, rtol=1e-8, atol=1e-10)


def test_simulate_matches_oracle(sbv, orc):
    rng = np.random.default_rng(3)
    mean = rng.normal(size=257)
    var = rng.uniform(0.0, 2.0, size=257)
    var[5] = 0.0
    h = sbv.Handle()
    g = h.simulate(mean, var, 1000, 11, 0.95)
    o = orc.simulate(mean, var, 1000, 11, 0.95)
    for a, b in zip(g, o):
        np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-13)


def test_predict_cfg2_shape_sampled(sbv, orc):
    """Training set of the bench shape (n=1M, d=10, bs=100, m=200), 50k test
    points, bs_pred=10, m_pred=200: structure in full, conditioning sets and
    mean / variance on 30 sampled test blocks."""
    c = si.CONFIGS["cfg2"]
    n, d = c["n"], c["d"]
    X = si.make_X(n, d, seed=1)
    y = si.make_y(X, seed=2)
    Xs = si.make_X(50_000, d, seed=3)
    sc = si.default_scale(d)
    theta = si.default_theta(d, nu=2.5, tau2=1e-4)
    import torch
    h = sbv.prepare(torch.from_numpy(X).cuda(), c["bs"], c["m"], sc)
    mean, var = h.predict(Xs, 10, 200, y, theta)
    anc, bo, off, perm, nbr, cnt = h.prediction_structure()
    ns = Xs.shape[0]
    k = orc.num_blocks(ns, 10)
    np.testing.assert_array_equal(anc, orc.anchors(ns, k, 3))
    St, S = orc.scale(Xs, sc), orc.scale(X, sc)
    np.testing.assert_array_equal(bo, orc.rac(St, anc))
    po, oo = orc.layout(bo, k)
    np.testing.assert_array_equal(perm, po)
    np.testing.assert_array_equal(off, oo)
    C = orc.centroids(St, perm, off)
    rng = np.random.default_rng(0)
    for t in rng.choice(k, 30, replace=False):
        J = orc.knn_pred(S, C[t], 200)
        np.testing.assert_array_equal(nbr[t, :cnt[t]], J)
        B = perm[off[t]:off[t + 1]]
        mo, vo = orc.predict_block(X, y, Xs, J, B, theta)
        assert np.abs(mean[B] - mo).max() <= 1e-9 * max(1.0, np.abs(y).max())
        assert np.abs(var[B] - vo).max() <= 1e-9 * (theta[0] + theta[d + 2])


def test_predict_and_simulate_argument_errors(sbv):
    X = si.make_X(500, 3, seed=1)
    y = si.make_y(X, seed=2)
    theta = si.default_theta(3, nu=2.5)
    h = sbv.Handle()
    with pytest.raises(sbv.SBVError) as e:  # not prepared
        h.predict(X[:10], 2, 10, y, theta)
    assert e.value.code == 7
    h = sbv.prepare(X, 10, 20, si.default_scale(3))
    with pytest.raises(sbv.SBVError) as e:
        h.predict(X[:10], 0, 10, y, theta)  # bs_pred < 1
    assert e.value.code == 1
    with pytest.raises(sbv.SBVError) as e:
        h.predict(X[:10], 2, 2000, y, theta)  # m_pred beyond the grid kNN
    assert e.value.code == 5
    Xs = X[:10].copy()
    Xs[2, 1] = np.inf
    with pytest.raises(sbv.SBVError) as e:
        h.predict(Xs, 2, 10, y, theta)
    assert e.value.code == 1
    with pytest.raises(sbv.SBVError) as e:
        h.simulate(np.zeros(3), np.array([1.0, -0.5, 1.0]), 100, 1)  # negative variance
    assert e.value.code == 1
    with pytest.raises(sbv.SBVError) as e:
        h.simulate(np.zeros(3), np.ones(3), 1, 1)  # n_sim < 2
    assert e.value.code == 1


def test_predict_general_nu(sbv, orc):
    """N2 x N3: prediction through the K_nu covariance path."""
    n, d = 2000, 3
    X = si.make_X(n, d, seed=61)
    y = si.make_y(X, seed=62)
    Xs = si.make_X(300, d, seed=63)
    sc = si.default_scale(d)
    theta = si.default_theta(d, nu=1.2, tau2=1e-3)
    h = sbv.prepare(X, 20, 40, sc)
    check(h, orc, X, y, Xs, 5, 30, theta, sc)
