"""Pins of the CPU oracle (oracle/) to things other than itself.

Every check here is independent of oracle arithmetic: published test vectors,
scipy's Bessel K_nu, the dense Eq.1 likelihood (numpy Cholesky), explicit-inverse
Gaussian conditionals, brute-force search on exactly-representable lattice data,
closed forms for tiny n, a variance scaling law and the KL invariant of Eq.4.
A dropped term, a wrong sign/index or a transposed operand anywhere in
oracle/sbv_oracle.c fails at least one of them.
"""
import math
import os

import numpy as np
import pytest
from scipy import special, stats

import sbv_inputs as si

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# --------------------------------------------------------------- independent helpers
def matern_bessel(r, sigma2, nu):
    """Eq.6 evaluated with scipy's modified Bessel K_nu, r>0."""
    r = np.asarray(r, dtype=np.float64)
    out = np.empty_like(r)
    pos = r > 0
    out[pos] = sigma2 * 2.0 ** (1 - nu) / special.gamma(nu) * r[pos] ** nu * special.kv(nu, r[pos])
    out[~pos] = sigma2  # r -> 0 limit of 2^{1-nu}/Gamma(nu) r^nu K_nu(r) is 1
    return out


def dense_cov(X, theta):
    """Sigma_theta of Eq.1 built from Eq.5 + Eq.6 via scipy Bessel; nugget on the diagonal."""
    d = X.shape[1]
    beta = theta[1:1 + d]
    Z = X / beta
    D = np.sqrt(((Z[:, None, :] - Z[None, :, :]) ** 2).sum(-1))
    K = matern_bessel(D, theta[0], theta[d + 1])
    return K + theta[d + 2] * np.eye(X.shape[0])


def dense_loglik(X, y, theta):
    """Eq.1 via numpy Cholesky."""
    S = dense_cov(X, theta)
    L = np.linalg.cholesky(S)
    z = np.linalg.solve(L, y)
    n = X.shape[0]
    return -0.5 * n * math.log(2 * math.pi) - np.log(np.diag(L)).sum() - 0.5 * z @ z


def rand_theta(d, nu, tau2, rng, lo=0.3, hi=1.5):
    return np.array([1.3, *(rng.uniform(lo, hi, d)), nu, tau2])


# --------------------------------------------------------------- O2 anchors / zeta
def test_splitmix64_published_vectors(orc):
    # tests/golden/splitmix64_seed0.txt: the reference splitmix64 generator's
    # first outputs for seed 0 (Q9 reading of "Randomly reorder").
    with open(os.path.join(GOLDEN, "splitmix64_seed0.txt")) as f:
        vals = [int(line.split()[1], 16) for line in f if line.strip() and not line.startswith("#")]
    assert len(vals) >= 3
    for i, v in enumerate(vals):
        assert orc.splitmix64(0, i) == v


def test_anchor_selection_is_k_smallest_keys(orc):
    n, k, seed = 5000, 137, 11
    a = orc.anchors(n, k, seed)
    keys = np.array([orc.splitmix64(seed, i) for i in range(n)], dtype=np.uint64)
    order = np.lexsort((np.arange(n), keys))  # by key, then index
    np.testing.assert_array_equal(a, order[:k])
    assert len(set(a.tolist())) == k


@pytest.mark.parametrize("n,bs,k", [(100, 10, 10), (105, 10, 11), (104, 10, 10), (5, 10, 1), (7, 1, 7), (1, 1, 1)])
def test_num_blocks_round(orc, n, bs, k):
    assert orc.num_blocks(n, bs) == k


# --------------------------------------------------------------- O1 / O7 kernel
def test_scaled_distance_spec_examples(orc):
    # S:52-54 (Eq.5): identical points -> 0; d=1 (0.1 vs 0, beta .05) -> 2; d=2 -> sqrt(13)
    assert orc.scaled_distance([0.3, 0.7], [0.3, 0.7], [0.2, 0.5]) == 0.0
    assert orc.scaled_distance([0.1], [0.0], [0.05]) == pytest.approx(2.0, rel=1e-15)
    assert orc.scaled_distance([0.3, 0.4], [0.0, 0.0], [0.1, 0.2]) == pytest.approx(math.sqrt(13), rel=1e-15)


def test_scale_divides(orc):
    X = si.make_X(50, 4, seed=5)
    s = np.array([0.5, 2.0, 0.25, 3.0])
    np.testing.assert_array_equal(orc.scale(X, s), X / s)  # IEEE division, elementwise


@pytest.mark.parametrize("nu", [0.5, 1.5, 2.5, 3.5])
def test_matern_closed_form_equals_bessel(orc, nu):
    r = np.concatenate([np.linspace(1e-6, 0.1, 50), np.linspace(0.1, 30, 300)])
    ref = matern_bessel(r, 1.7, nu)
    got = np.array([orc.matern(x, 1.7, nu) for x in r])
    np.testing.assert_allclose(got, ref, rtol=2e-13, atol=1e-300)


@pytest.mark.parametrize("nu", [0.5, 1.5, 2.5, 3.5])
def test_matern_limits_and_decay(orc, nu):
    assert orc.matern(0.0, 1.0, nu) == 1.0
    # r=0, sigma2=1, tau2=0.25 -> 1.25 (nugget only on the same point)
    th = np.array([1.0, 0.3, nu, 0.25])
    assert orc.kernel([0.4], [0.4], th, True) == 1.25
    assert orc.kernel([0.4], [0.4], th, False) == 1.0
    vals = [orc.matern(r, 1.0, nu) for r in np.linspace(0, 40, 400)]
    assert all(a >= b for a, b in zip(vals, vals[1:]))
    assert vals[-1] < 1e-12


def test_unsupported_nu_is_nan(orc):
    assert math.isnan(orc.matern(1.0, 1.0, 0.0))
    assert math.isnan(orc.matern(1.0, 1.0, -1.0))
    assert math.isnan(orc.matern(1.0, 1.0, 25.0))


@pytest.mark.parametrize("nu", [0.2, 0.5, 0.75, 1.0, 1.3, 2.0, 2.5, 3.7, 6.4])
def test_besselk_integral_equals_scipy(orc, nu):
    """N3: the oracle's K_nu (trapezoid on the cosh integral) = scipy.special.kv."""
    for r in [1e-6, 1e-3, 0.05, 0.3, 1.0, 1.99, 2.01, 5.0, 17.0, 80.0, 300.0]:
        ref = special.kv(nu, r)
        assert abs(orc.besselk(nu, r) - ref) <= 1e-13 * ref, (nu, r)


@pytest.mark.parametrize("nu", [0.3, 1.0, 2.0, 4.25])
def test_general_nu_matern_equals_bessel(orc, nu):
    """N3: Eq.6 for non-half-integer nu = the scipy Bessel form; r=0 limit."""
    for r in [1e-8, 1e-4, 0.01, 0.5, 1.0, 3.0, 10.0, 50.0]:
        ref = matern_bessel(np.array(r), 1.7, nu)
        assert abs(orc.matern(r, 1.7, nu) - ref) <= 1e-12 * max(ref, 1e-300), (nu, r)
    assert orc.matern(0.0, 1.7, nu) == 1.7
    # continuity across a half-integer: nu -> 1.5 matches the closed form
    assert abs(orc.matern(0.8, 1.0, 1.5 + 1e-9) - orc.matern(0.8, 1.0, 1.5)) < 1e-8


# --------------------------------------------------------------- O8/O9 likelihood
@pytest.mark.parametrize("nu", [1.5, 2.5, 3.5])
@pytest.mark.parametrize("bs", [1, 10])
def test_full_conditioning_equals_dense(orc, nu, bs):
    """S:577 acceptance #1 / chain rule P:187-190: m >= n => Eq.2 == Eq.1."""
    rng = np.random.default_rng(100 + bs)
    n, d = 300, 10
    X = si.make_X(n, d, seed=21)
    y = si.make_y(X, seed=22, kind="iid")
    theta = rand_theta(d, nu, 1e-3, rng, 0.8, 3.0)
    P = orc.prepare(X, bs, n - 1, theta[1:1 + d], seed=3)
    ll = orc.loglik(X, y, P["perm"], P["off"], P["nbr"], P["cnt"], theta)
    ref = dense_loglik(X, y, theta)
    assert abs(ll - ref) <= 1e-9 * abs(ref)


def test_single_block_equals_dense(orc):
    """bs = n => one block, no neighbours => Eq.1."""
    n, d = 150, 3
    X = si.make_X(n, d, seed=31)
    y = si.make_y(X, seed=32)
    theta = np.array([0.9, 0.3, 0.6, 0.2, 2.5, 1e-3])
    P = orc.prepare(X, n, 40, theta[1:4], seed=1)
    assert P["k"] == 1 and P["cnt"][0] == 0
    ll = orc.loglik(X, y, P["perm"], P["off"], P["nbr"], P["cnt"], theta)
    assert abs(ll - dense_loglik(X, y, theta)) <= 1e-10 * abs(ll)


@pytest.mark.parametrize("nu", [0.5, 3.5])
def test_block_terms_equal_explicit_inverse_conditionals(orc, nu):
    """each block term equals log N(y_B; mu, Sigma) with the conditional
    mean/covariance formed by explicit inverses (P:177-183 applied per block)."""
    n, d, bs, m = 40, 3, 5, 10
    X = si.make_X(n, d, seed=41)
    y = si.make_y(X, seed=42, kind="iid")
    theta = np.array([1.1, 0.4, 0.7, 0.3, nu, 1e-2])
    P = orc.prepare(X, bs, m, theta[1:4], seed=7)
    ll, terms, quads, logdets = orc.loglik(X, y, P["perm"], P["off"], P["nbr"], P["cnt"], theta,
                                           return_terms=True)
    Sig = dense_cov(X, theta)
    ref_total = 0.0
    for t in range(P["k"]):
        B = P["perm"][P["off"][t]:P["off"][t + 1]]
        J = P["nbr"][t, :P["cnt"][t]]
        if len(J):
            W = Sig[np.ix_(B, J)] @ np.linalg.inv(Sig[np.ix_(J, J)])
            mu = W @ y[J]
            C = Sig[np.ix_(B, B)] - W @ Sig[np.ix_(J, B)]
        else:
            mu, C = np.zeros(len(B)), Sig[np.ix_(B, B)]
        ref = stats.multivariate_normal(mean=mu, cov=C).logpdf(y[B])
        assert abs(terms[t] - ref) <= 1e-10 * max(1.0, abs(ref)), t
        ref_total += ref
    assert abs(ll - ref_total) <= 1e-10 * abs(ref_total)


def test_n1_closed_form(orc):
    # n=1 => -1/2 log 2pi - 1/2 log s - y^2/(2s), s = sigma2 + tau2
    X = np.array([[0.3, 0.1]])
    for yv, s2, t2 in [(0.0, 1.0, 0.0), (1.0, 1.0, 0.0), (-0.7, 2.0, 0.5)]:
        th = np.array([s2, 0.2, 0.2, 2.5, t2])
        P = orc.prepare(X, 1, 5, th[1:3], seed=0)
        ll = orc.loglik(X, np.array([yv]), P["perm"], P["off"], P["nbr"], P["cnt"], th)
        s = s2 + t2
        assert ll == pytest.approx(-0.5 * math.log(2 * math.pi) - 0.5 * math.log(s) - yv * yv / (2 * s), rel=1e-14)


def test_bs1_m0_is_sum_of_univariate_normals(orc):
    n = 30
    X = si.make_X(n, 2, seed=51)
    y = si.make_y(X, seed=52, kind="iid")
    th = np.array([1.4, 0.3, 0.3, 1.5, 0.1])
    P = orc.prepare(X, 1, 0, th[1:3], seed=4)
    ll = orc.loglik(X, y, P["perm"], P["off"], P["nbr"], P["cnt"], th)
    ref = stats.norm(0, math.sqrt(1.5)).logpdf(y).sum()
    assert ll == pytest.approx(ref, rel=1e-13)


def test_n2_bs1_m1_is_bivariate_normal(orc):
    X = np.array([[0.1, 0.2], [0.3, 0.25]])
    y = np.array([0.4, -0.3])
    th = np.array([1.2, 0.5, 0.4, 2.5, 0.05])
    P = orc.prepare(X, 1, 1, th[1:3], seed=9)
    ll = orc.loglik(X, y, P["perm"], P["off"], P["nbr"], P["cnt"], th)
    ref = stats.multivariate_normal(mean=[0, 0], cov=dense_cov(X, th)).logpdf(y)
    assert ll == pytest.approx(ref, rel=1e-13)


def test_variance_scaling_law(orc):
    """l_t(c s2, c t2; y) = l_t(s2, t2; y / sqrt c) - (bs_t/2) log c, block by block."""
    n, d, c = 200, 4, 3.7
    X = si.make_X(n, d, seed=61)
    y = si.make_y(X, seed=62, kind="iid")
    th = np.array([1.0, 0.5, 0.4, 0.9, 1.2, 2.5, 1e-3])
    P = orc.prepare(X, 8, 20, th[1:5], seed=5)
    thc = th.copy()
    thc[0] *= c
    thc[-1] *= c
    _, t1, _, _ = orc.loglik(X, y, P["perm"], P["off"], P["nbr"], P["cnt"], thc, return_terms=True)
    _, t2, _, _ = orc.loglik(X, y / math.sqrt(c), P["perm"], P["off"], P["nbr"], P["cnt"], th,
                             return_terms=True)
    bsz = np.diff(P["off"])
    np.testing.assert_allclose(t1, t2 - 0.5 * bsz * math.log(c), rtol=1e-11, atol=1e-11)


def test_kl_nonnegative_and_monotone_in_m(orc):
    """Eq.4: KL = l0(theta;0) - la(theta;0) >= 0; neighbour sets are
    nested in m so KL is nonincreasing in m and vanishes at full conditioning."""
    n, d = 400, 10
    X = si.make_X(n, d, seed=71)
    th = si.default_theta(d, nu=2.5, tau2=1e-3, beta=(0.25, 0.25) + (5.0,) * 8)
    y0 = np.zeros(n)
    l0 = dense_loglik(X, y0, th)
    kls = []
    for m in [0, 5, 10, 20, 40, 80, n]:
        P = orc.prepare(X, 10, m, th[1:1 + d], seed=3)
        kls.append(l0 - orc.loglik(X, y0, P["perm"], P["off"], P["nbr"], P["cnt"], th))
    assert all(k >= -1e-8 for k in kls)
    assert all(a >= b - 1e-8 for a, b in zip(kls, kls[1:]))
    assert abs(kls[-1]) < 1e-8 and kls[0] > 1.0


def test_not_pd_reports_block_and_stage(orc):
    """Duplicate points with tau2 = 0 are singular (Q17): reported, not jittered."""
    X = si.make_X(60, 2, seed=81, kind="duplicates")
    th = np.array([1.0, 0.3, 0.3, 2.5, 0.0])
    P = orc.prepare(X, 60, 0, th[1:3], seed=1)  # one block holds both copies
    with pytest.raises(orc.NotPD) as e:
        orc.loglik(X, np.zeros(60), P["perm"], P["off"], P["nbr"], P["cnt"], th)
    assert e.value.block == 0 and e.value.stage == 2
    # conditioning set holding both copies -> stage 1
    P = orc.prepare(X, 1, 59, th[1:3], seed=1)
    with pytest.raises(orc.NotPD) as e:
        orc.loglik(X, np.zeros(60), P["perm"], P["off"], P["nbr"], P["cnt"], th)
    assert e.value.stage in (1, 2)


# --------------------------------------------------------------- O3-O6 clustering / kNN
def _np_d2(a, B):
    return ((B - a) ** 2).sum(-1)


def _fma_chain_d2(a, b):
    """dist2 by the definition of IEEE fma (Q14): t = RN(a_j - b_j),
    acc = RN(t*t + acc) with the product and sum exact (Fractions), in
    dimension order.  int/int true division in CPython is correctly rounded."""
    from fractions import Fraction
    acc = 0.0
    for x, z in zip(a, b):
        t = float(x) - float(z)
        q = Fraction(t) * Fraction(t) + Fraction(acc)
        acc = q.numerator / q.denominator
    return acc


def test_rac_and_knn_exact_on_lattice(orc):
    """Lattice coordinates k/8 with power-of-two scales: every difference, square
    and partial sum is exact, so numpy's arithmetic equals the fma chain and the
    brute-force argmin / lexicographic sort is the exact reference (massive ties
    exercise the index tie rules Q8/Q13)."""
    n, d, bs, m = 600, 3, 6, 25
    X = si.make_X(n, d, seed=91, kind="lattice")
    scale = np.array([0.5, 1.0, 2.0])
    P = orc.prepare(X, bs, m, scale, seed=13)
    S = X / scale
    anc = P["anchors"]
    # RAC: first minimum over anchor rank; anchors keep their own block
    for i in range(n):
        dd = _np_d2(S[i], S[anc])
        want = np.argmin(dd)
        if i in set(anc.tolist()):
            want = int(np.where(anc == i)[0][0])
        assert P["block_of"][i] == want
    # layout
    for t in range(P["k"]):
        mem = P["perm"][P["off"][t]:P["off"][t + 1]]
        assert np.all(np.diff(mem) > 0) and np.all(P["block_of"][mem] == t)
    # centroids: exact means here too (sums of k/16 values / size) up to one rounding
    for t in range(P["k"]):
        mem = P["perm"][P["off"][t]:P["off"][t + 1]]
        np.testing.assert_allclose(P["C"][t], S[mem].mean(0), rtol=1e-15, atol=1e-15)
    # kNN over strictly earlier blocks, full lexicographic sort (dist2, index);
    # centroids are not lattice points, so distances use the exact fma definition
    for t in range(0, P["k"], 3):
        adm = P["perm"][:P["off"][t]]
        dd = np.array([_fma_chain_d2(P["C"][t], S[i]) for i in adm])
        order = adm[np.lexsort((adm, dd))][:m]
        np.testing.assert_array_equal(P["nbr"][t, :P["cnt"][t]], order)
        assert P["cnt"][t] == min(m, P["off"][t])


@pytest.mark.parametrize("d,m", [(2, 10), (5, 60), (10, 200)])
def test_knn_matches_bruteforce_random(orc, d, m):
    """exact kNN equals a full-sort brute force.  Random data: numpy's
    non-fma distances may differ from the fma chain in the last ulp, so the
    comparison is exact outside near-ties (|delta| < 1e-13 relative)."""
    n = 3000
    X = si.make_X(n, d, seed=200 + d)
    P = orc.prepare(X, 20, m, np.full(d, 0.3), seed=17)
    S = X / 0.3
    for t in range(0, P["k"], 7):
        adm = P["perm"][:P["off"][t]]
        dd = _np_d2(P["C"][t], S[adm])
        order = adm[np.lexsort((adm, dd))][:m]
        got = P["nbr"][t, :P["cnt"][t]]
        if not np.array_equal(got, order):
            dg = _np_d2(P["C"][t], S[got])
            do = _np_d2(P["C"][t], S[order])
            np.testing.assert_allclose(dg, do, rtol=1e-13)
        assert np.all(np.isin(got, adm))


def test_rac_extremes(orc):
    X = si.make_X(50, 3, seed=3)
    P = orc.prepare(X, 1, 3, np.ones(3), seed=2)  # k = n -> singletons
    assert P["k"] == 50 and np.all(np.diff(P["off"]) == 1)
    P = orc.prepare(X, 50, 3, np.ones(3), seed=2)  # k = 1 -> one block
    assert P["k"] == 1 and P["off"][1] == 50 and P["cnt"][0] == 0


def test_rac_random_is_nearest_anchor(orc):
    n, d = 2000, 10
    X = si.make_X(n, d, seed=301)
    sc = si.default_scale(d)
    P = orc.prepare(X, 20, 10, sc, seed=3)
    S = X / sc
    anc = P["anchors"]
    for i in range(0, n, 13):
        dd = _np_d2(S[i], S[anc])
        got = P["block_of"][i]
        assert dd[got] <= dd.min() * (1 + 1e-13)


# --------------------------------------------------------------- round-2 pins
def test_centroids_left_to_right_order(orc):
    """O5 (Alg.4 line 6): c_t = (((0 + s_i1) + s_i2) + ...) / |b|
    with members ascending, bit for bit.  The data mixes magnitudes so that the
    summation order changes the rounding: a reversed (or pairwise) sum fails."""
    rng = np.random.default_rng(123)
    n, d = 3000, 4
    X = rng.random((n, d)) * 10.0 ** rng.integers(-6, 7, size=(n, d))
    scale_ = np.array([0.3, 1.7, 0.05, 3.1])
    S = orc.scale(X, scale_)
    k = 37
    bo = rng.integers(0, k, size=n).astype(np.int32)
    perm, off = orc.layout(bo, k)
    C = orc.centroids(S, perm, off)
    differs = 0
    for t in range(k):
        members = perm[off[t]:off[t + 1]]
        assert list(members) == sorted(members)  # O4: ascending original index
        for j in range(d):
            acc = 0.0
            for i in members:  # Python floats are IEEE binary64: one rounding per add
                acc = acc + float(S[i, j])
            assert C[t, j] == acc / len(members), (t, j)
            rev = 0.0
            for i in members[::-1]:
                rev = rev + float(S[i, j])
            differs += (rev / len(members)) != C[t, j]
    assert differs > 0  # the pin can tell the orders apart on this data


def test_block_term_at_equals_loglik_terms(orc):
    """orc_block_term_at (used by the sampled cfg2/cfg4 parity tests) returns the
    same term as orc_loglik's per-block output (bitwise: same arithmetic), and
    that term equals the explicit-inverse Gaussian conditional."""
    n, d, bs, m = 600, 4, 12, 25
    X = si.make_X(n, d, seed=141)
    y = si.make_y(X, seed=142)
    theta = np.array([1.2, 0.3, 0.5, 0.9, 0.4, 2.5, 1e-3])
    P = orc.prepare(X, bs, m, theta[1:1 + d], seed=9)
    ll, terms, quads, logdets = orc.loglik(X, y, P["perm"], P["off"], P["nbr"], P["cnt"], theta,
                                           return_terms=True)
    Sig = dense_cov(X, theta)
    for t in list(range(0, P["k"], 7)) + [P["k"] - 1]:
        to, qo, lo = orc.block_term_at(X, y, P["perm"], P["off"], P["nbr"], P["cnt"], t, theta)
        assert (to, qo, lo) == (terms[t], quads[t], logdets[t]), t
        B = P["perm"][P["off"][t]:P["off"][t + 1]]
        J = P["nbr"][t, :P["cnt"][t]]
        if len(J):
            W = Sig[np.ix_(B, J)] @ np.linalg.inv(Sig[np.ix_(J, J)])
            mu, C = W @ y[J], Sig[np.ix_(B, B)] - W @ Sig[np.ix_(J, B)]
        else:
            mu, C = np.zeros(len(B)), Sig[np.ix_(B, B)]
        ref = stats.multivariate_normal(mean=mu, cov=C).logpdf(y[B])
        assert abs(to - ref) <= 1e-9 * max(1.0, abs(ref)), t
