"""GPU parity: libsbv (CUDA, through the C ABI) against the CPU oracle.

Bar (BASELINE.json north_star): block/neighbour indices bit-exact, per-block
terms within 1e-10 relative, the log-likelihood within 1e-9 relative
(Q18 relative base).  Inputs are seeded and synthetic (sbv_inputs).
"""
import math

import numpy as np
import pytest

import sbv_inputs as si

pytestmark = pytest.mark.gpu

TOL_LL = 1e-9
TOL_TERM = 1e-10


@pytest.fixture(scope="module")
def sbv():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2504_12004_b200 as p
    from paper_2504_12004_b200 import build
    build.build()
    return p


def run_both(sbv, orc, X, y, bs, m, scale, theta, seed=3, device=True):
    import torch
    Xt = torch.from_numpy(X).cuda() if device else X
    yt = torch.from_numpy(y).cuda() if device else y
    h = sbv.prepare(Xt, bs, m, scale, seed=seed)
    P = orc.prepare(X, bs, m, scale, seed)
    return h, P, Xt, yt


def check_indices(h, P):
    np.testing.assert_array_equal(h.anchors(), P["anchors"])
    bo, off, perm, C = h.blocks()
    np.testing.assert_array_equal(bo, P["block_of"])
    np.testing.assert_array_equal(off, P["off"])
    np.testing.assert_array_equal(perm, P["perm"])
    np.testing.assert_array_equal(C, P["C"])  # bit-exact centroids (same summation order)
    nbr, cnt = h.neighbors()
    np.testing.assert_array_equal(cnt, P["cnt"])
    np.testing.assert_array_equal(nbr, P["nbr"])


def check_terms(h, orc, X, y, yt, P, theta):
    ll_o, terms_o, quads_o, logdets_o = orc.loglik(X, y, P["perm"], P["off"], P["nbr"], P["cnt"],
                                                    theta, return_terms=True)
    terms, quads, logdets = h.block_terms(yt, theta)
    # DESIGN.md Q18: relative to the term's own magnitude, guarded against
    # cancellation between its parts (-1/2 quad, -1/2 logdet, -bs/2 log 2pi)
    bsz = np.diff(P["off"])
    base = np.maximum(np.abs(terms_o),
                      0.5 * (np.abs(quads_o) + np.abs(logdets_o)) + 0.5 * bsz * math.log(2 * math.pi))
    rel = np.abs(terms - terms_o) / base
    assert rel.max() <= TOL_TERM, (rel.max(), int(rel.argmax()))
    ll = h.loglik(yt, theta)
    den = max(abs(ll_o), np.abs(terms_o).sum())
    assert abs(ll - ll_o) <= TOL_LL * den, (ll, ll_o)
    return ll, ll_o


@pytest.mark.parametrize("d,bs,m,nu", [
    (10, 20, 60, 2.5),   # cfg1 shape, reduced n
    (10, 10, 30, 3.5),   # paper's nu, bs=10
    (2, 7, 13, 0.5),
    (5, 33, 90, 1.5),
    (3, 1, 5, 2.5),      # bs = 1 (SV degenerate)
    (10, 50, 0, 2.5),    # m = 0: marginal block terms only
])
def test_parity_small(sbv, orc, d, bs, m, nu):
    n = 3000
    X = si.make_X(n, d, seed=10 + d)
    y = si.make_y(X, seed=20 + d)
    scale = si.default_scale(d)
    theta = si.default_theta(d, nu=nu, tau2=1e-4)
    h, P, Xt, yt = run_both(sbv, orc, X, y, bs, m, scale, theta)
    check_indices(h, P)
    check_terms(h, orc, X, y, yt, P, theta)


@pytest.mark.parametrize("d", [1, 20, 64])
def test_parity_dimension_edges(sbv, orc, d):
    """d = 1 and the generic (d > 16) coordinate paths of RAC, kNN and H8, up to SBV_MAX_D."""
    n = 1500
    X = si.make_X(n, d, seed=100 + d)
    y = si.make_y(X, seed=200 + d)
    scale = np.linspace(0.5, 2.0, d)
    theta = np.array([1.1, *np.linspace(0.6, 3.0, d), 1.5, 1e-3])
    h, P, Xt, yt = run_both(sbv, orc, X, y, 15, 35, scale, theta)
    check_indices(h, P)
    check_terms(h, orc, X, y, yt, P, theta)


def test_parity_large_blocks_multi_pass(sbv, orc):
    """N_t = m + bs up to ~700 rows: several 256-row passes per panel, ragged tails."""
    n, d, bs, m = 4000, 4, 300, 350
    X = si.make_X(n, d, seed=5)
    y = si.make_y(X, seed=6)
    scale = np.array([0.2, 0.3, 1.0, 2.0])
    theta = np.array([1.3, 0.2, 0.3, 1.0, 2.0, 2.5, 1e-3])
    h, P, Xt, yt = run_both(sbv, orc, X, y, bs, m, scale, theta)
    check_indices(h, P)
    check_terms(h, orc, X, y, yt, P, theta)
    assert h.stats()["max_N"] > 600


def test_parity_lattice_ties(sbv, orc):
    """Exactly representable lattice data: massive distance ties exercise the
    index tie rules of RAC (lowest anchor rank) and kNN (lowest index)."""
    n, d = 2500, 3
    X = si.make_X(n, d, seed=77, kind="lattice")
    y = si.make_y(X, seed=78)
    scale = np.array([0.5, 1.0, 2.0])
    theta = np.array([1.0, 0.5, 1.0, 2.0, 2.5, 1e-2])
    h, P, Xt, yt = run_both(sbv, orc, X, y, 12, 40, scale, theta)
    check_indices(h, P)


def test_full_conditioning_matches_dense_via_gpu(sbv, orc):
    """m >= n: the GPU block-Vecchia likelihood equals the exact Eq.1 likelihood."""
    from tests.test_oracle_pins import dense_loglik
    import torch
    n, d = 300, 10
    X = si.make_X(n, d, seed=21)
    y = si.make_y(X, seed=22, kind="iid")
    theta = np.array([1.3, *np.linspace(0.8, 3.0, d), 2.5, 1e-3])
    h = sbv.prepare(torch.from_numpy(X).cuda(), 10, n - 1, theta[1:1 + d])
    ll = h.loglik(torch.from_numpy(y).cuda(), theta)
    ref = dense_loglik(X, y, theta)
    assert abs(ll - ref) <= 1e-9 * abs(ref)


def test_host_and_device_pointers_agree(sbv, orc):
    n, d = 1500, 6
    X = si.make_X(n, d, seed=31)
    y = si.make_y(X, seed=32)
    theta = si.default_theta(d, nu=2.5)
    import torch
    h1 = sbv.prepare(X, 15, 40, si.default_scale(d))
    h2 = sbv.prepare(torch.from_numpy(X).cuda(), 15, 40, si.default_scale(d))
    a = h1.loglik(y, theta)
    b = h2.loglik(torch.from_numpy(y).cuda(), theta)
    assert a == b  # same kernels, same order: bitwise
    assert h1.loglik(y, theta) == a  # repeatable


def test_not_pd_reports_lowest_block_and_stage(sbv, orc):
    X = si.make_X(400, 2, seed=81, kind="duplicates")
    theta = np.array([1.0, 0.3, 0.3, 2.5, 0.0])
    y = np.zeros(400)
    h = sbv.prepare(X, 400, 0, theta[1:3])  # one block containing both copies
    with pytest.raises(sbv.SBVError) as e:
        h.loglik(y, theta)
    assert e.value.code == 4 and e.value.block == 0 and e.value.stage == 2
    # full conditioning: the later copy's conditioning set holds the earlier copy
    P = orc.prepare(X, 1, 399, theta[1:3], 3)
    with pytest.raises(orc.NotPD) as eo:
        orc.loglik(X, y, P["perm"], P["off"], P["nbr"], P["cnt"], theta)
    h = sbv.prepare(X, 1, 399, theta[1:3])
    with pytest.raises(sbv.SBVError) as e:
        h.loglik(y, theta)
    assert e.value.block == eo.value.block and e.value.stage == eo.value.stage


def test_argument_errors(sbv):
    X = si.make_X(100, 3, seed=1)
    with pytest.raises(sbv.SBVError) as e:
        sbv.prepare(X, 0, 5, np.ones(3))
    assert e.value.code == 1
    with pytest.raises(sbv.SBVError):
        sbv.prepare(X, 10, 5, np.array([1.0, -1.0, 1.0]))
    Xn = X.copy()
    Xn[3, 1] = np.nan
    with pytest.raises(sbv.SBVError):
        sbv.prepare(Xn, 10, 5, np.ones(3))
    h = sbv.prepare(X, 10, 5, np.ones(3))
    with pytest.raises(sbv.SBVError) as e:
        h.loglik(np.zeros(100), np.array([1.0, 1, 1, 1, 25.0, 0.0]))  # nu > 20 unsupported
    assert e.value.code == 5
    with pytest.raises(sbv.SBVError) as e:
        h.loglik(np.zeros(100), np.array([-1.0, 1, 1, 1, 2.5, 0.0]))
    assert e.value.code == 1


def test_grid_search_equals_brute_force(sbv, monkeypatch):
    """The grid-filtered RAC / multi-level kNN against the
    exhaustive kernels (SBV_GRID=0, oracle-checked at small n) at a size with
    several prefix levels: identical partitions, neighbours and likelihood."""
    import torch
    n, d, bs, m = 300_000, 10, 30, 100
    X = torch.from_numpy(si.make_X(n, d, seed=41)).cuda()
    y = torch.from_numpy(si.make_y(X.cpu().numpy(), seed=42)).cuda()
    sc = si.default_scale(d)
    theta = si.default_theta(d, nu=1.5, tau2=1e-4)
    hg = sbv.prepare(X, bs, m, sc)
    monkeypatch.setenv("SBV_GRID", "0")
    hb = sbv.prepare(X, bs, m, sc)
    np.testing.assert_array_equal(hg.anchors(), hb.anchors())
    for a, b in zip(hg.blocks(), hb.blocks()):
        np.testing.assert_array_equal(a, b)
    for a, b in zip(hg.neighbors(), hb.neighbors()):
        np.testing.assert_array_equal(a, b)
    assert hg.loglik(y, theta) == hb.loglik(y, theta)


def test_knn_shared_query_mode_equals_warp_mode(sbv, monkeypatch):
    """Few queries run with the CTA's warps sharing each query (SBV_KNN_QW=4);
    the neighbour sets must equal the one-warp-per-query kernel's."""
    import torch
    n, d, bs, m = 200_000, 10, 100, 200
    X = torch.from_numpy(si.make_X(n, d, seed=44)).cuda()
    sc = si.default_scale(d)
    monkeypatch.setenv("SBV_KNN_QW", "4")
    h4 = sbv.prepare(X, bs, m, sc)
    monkeypatch.setenv("SBV_KNN_QW", "1")
    h1 = sbv.prepare(X, bs, m, sc)
    for a, b in zip(h4.neighbors(), h1.neighbors()):
        np.testing.assert_array_equal(a, b)


def test_cfg2_full_size_sampled(sbv, orc):
    """BASELINE.json configs[1] (n=1e6, d=10, bs=100, m=200) in the launch
    configuration bench.py times: anchors, layout and centroids in full,
    nearest-anchor assignment on 4,000 sampled points, the neighbour sets and
    block terms of 40 sampled blocks (every prefix level), and the total
    against the oracle's sum over the GPU's (sample-verified) structure."""
    import torch
    c = si.CONFIGS["cfg2"]
    n, d, bs, m = c["n"], c["d"], c["bs"], c["m"]
    X = si.make_X(n, d, seed=1)
    y = si.make_y(X, seed=2, kind="iid")
    sc = si.default_scale(d)
    theta = si.default_theta(d, nu=c["nu"], tau2=1e-4)
    h = sbv.prepare(torch.from_numpy(X).cuda(), bs, m, sc)
    k = orc.num_blocks(n, bs)
    anc = h.anchors()
    np.testing.assert_array_equal(anc, orc.anchors(n, k, 3))
    S = orc.scale(X, sc)
    bo, off, perm, C = h.blocks()
    rng = np.random.default_rng(7)
    smp = np.setdiff1d(rng.choice(n, 4000, replace=False), anc)
    # nearest anchor of sampled points: anchors first, so anchor rank r is row r
    bo_s = orc.rac(np.concatenate([S[anc], S[smp]]), np.arange(k, dtype=np.int32))[k:]
    np.testing.assert_array_equal(bo[smp], bo_s)
    perm_o, off_o = orc.layout(bo, k)
    np.testing.assert_array_equal(perm, perm_o)
    np.testing.assert_array_equal(off, off_o)
    np.testing.assert_array_equal(C, orc.centroids(S, perm, off))
    nbr, cnt = h.neighbors()
    # 40 blocks over the zeta order, log-spaced so every prefix level is hit
    ts = np.unique(np.concatenate([[0, 1, 2, k - 1],
                                   np.geomspace(3, k - 2, 36).astype(np.int64)]))
    for t in ts:
        ref = orc.knn_block(S, perm, off, C, int(t), m)
        assert cnt[t] == len(ref), t
        np.testing.assert_array_equal(nbr[t, :cnt[t]], ref, err_msg=f"block {t}")
    terms, quads, logdets = h.block_terms(torch.from_numpy(y).cuda(), theta)
    for t in ts:
        to, qo, lo = orc.block_term_at(X, y, perm, off, nbr, cnt, int(t), theta)
        b = max(abs(to), 0.5 * (abs(qo) + abs(lo)) + 0.5 * (off[t + 1] - off[t]) * math.log(2 * math.pi))
        assert abs(terms[t] - to) <= TOL_TERM * b, (t, terms[t], to)
    ll = h.loglik(torch.from_numpy(y).cuda(), theta)
    ll_o = orc.loglik(X, y, perm, off, nbr, cnt, theta)
    assert abs(ll - ll_o) <= TOL_LL * max(abs(ll_o), np.abs(terms).sum()), (ll, ll_o)


@pytest.mark.parametrize("nu", [0.3, 1.0, 2.0, 4.25])
def test_parity_general_nu(sbv, orc, nu):
    """non-half-integer smoothness through the K_nu path."""
    n, d = 2500, 5
    X = si.make_X(n, d, seed=90)
    y = si.make_y(X, seed=91)
    scale = si.default_scale(d)
    theta = si.default_theta(d, nu=nu, tau2=1e-3)
    h, P, Xt, yt = run_both(sbv, orc, X, y, 10, 40, scale, theta)
    check_terms(h, orc, X, y, yt, P, theta)


def test_cfg1_full_size(sbv, orc):
    """BASELINE.json configs[0]: n=20,000, d=10, bs=20, m=60, Matérn-5/2."""
    c = si.CONFIGS["cfg1"]
    X = si.make_X(c["n"], c["d"], seed=1)
    y = si.make_y(X, seed=2)
    theta = si.default_theta(c["d"], nu=c["nu"], tau2=1e-4)
    h, P, Xt, yt = run_both(sbv, orc, X, y, c["bs"], c["m"], si.default_scale(c["d"]), theta)
    check_indices(h, P)
    check_terms(h, orc, X, y, yt, P, theta)
