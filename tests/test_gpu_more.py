"""GPU parity, round 2: the remaining boundary calls, the H10 exchange
arithmetic on one device, the cfg4 shape, the brute-force kNN path (m > 960),
the caller-given block partition and an informational tau2 = 0 run.

Same bar as tests/test_gpu_parity.py (BASELINE.json north_star): indices
bit-exact, per-block terms within 1e-10 (Q18b base; the strict
|d ell_t| / |ell_t| is reported alongside), ell within 1e-9 relative.
"""
import ctypes
import json
import math
import os

import numpy as np
import pytest

import sbv_inputs as si

pytestmark = pytest.mark.gpu

TOL_LL = 1e-9
TOL_TERM = 1e-10
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REPORT = os.path.join(ROOT, "gpurun_out", "parity_report.jsonl")


@pytest.fixture(scope="module")
def sbv():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2504_12004_b200 as p
    from paper_2504_12004_b200 import build
    build.build()
    return p


def report(name, **kw):
    os.makedirs(os.path.dirname(REPORT), exist_ok=True)
    with open(REPORT, "a") as f:
        f.write(json.dumps({"test": name, **kw}) + "\n")


def term_errors(terms, terms_o, quads_o, logdets_o, bsz):
    base = np.maximum(np.abs(terms_o),
                      0.5 * (np.abs(quads_o) + np.abs(logdets_o)) + 0.5 * bsz * math.log(2 * math.pi))
    q18b = np.abs(terms - terms_o) / base
    strict = np.abs(terms - terms_o) / np.maximum(np.abs(terms_o), 1e-300)
    return q18b, strict


def compare_all(name, h, orc, X, y, yt, P, theta, tol_term=TOL_TERM, tol_ll=TOL_LL):
    ll_o, terms_o, quads_o, logdets_o = orc.loglik(X, y, P["perm"], P["off"], P["nbr"], P["cnt"],
                                                    theta, return_terms=True)
    terms, _, _ = h.block_terms(yt, theta)
    q18b, strict = term_errors(terms, terms_o, quads_o, logdets_o, np.diff(P["off"]))
    ll = h.loglik(yt, theta)
    den = max(abs(ll_o), np.abs(terms_o).sum())
    report(name, max_rel_term_q18b=float(q18b.max()), max_rel_term_strict=float(strict.max()),
           median_rel_term_strict=float(np.median(strict)), rel_ll=abs(ll - ll_o) / abs(ll_o),
           rel_ll_q18=abs(ll - ll_o) / den)
    assert q18b.max() <= tol_term, (q18b.max(), int(q18b.argmax()))
    assert abs(ll - ll_o) <= tol_ll * den, (ll, ll_o)
    return ll, ll_o


def test_north_star_entry_points_through_ctypes(sbv, orc):
    """sbv_prepare (north-star signature), sbv_prepare_ex and sbv_loglik_parts
    called directly through the C ABI on device buffers."""
    import torch
    L = sbv.lib()
    n, d, bs, m = 2000, 10, 20, 60
    X = si.make_X(n, d, seed=51)
    y = si.make_y(X, seed=52)
    scale = si.default_scale(d)
    theta = si.default_theta(d, nu=2.5, tau2=1e-4)
    Xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
    sc = np.ascontiguousarray(scale)
    th = np.ascontiguousarray(theta)
    P = orc.prepare(X, bs, m, scale, 3)
    ll_o = orc.loglik(X, y, P["perm"], P["off"], P["nbr"], P["cnt"], theta)
    h = ctypes.c_void_p()
    assert L.sbv_prepare(ctypes.c_void_p(Xd.data_ptr()), n, d, bs, m,
                         sc.ctypes.data_as(ctypes.c_void_p), ctypes.byref(h)) == 0
    ll = ctypes.c_double()
    assert L.sbv_loglik(h, ctypes.c_void_p(yd.data_ptr()), th.ctypes.data_as(ctypes.c_void_p),
                        ctypes.byref(ll)) == 0
    assert abs(ll.value - ll_o) <= TOL_LL * abs(ll_o)
    parts = np.zeros(4)
    assert L.sbv_loglik_parts(h, ctypes.c_void_p(yd.data_ptr()), th.ctypes.data_as(ctypes.c_void_p),
                              parts.ctypes.data_as(ctypes.c_void_p)) == 0
    assert parts[0] == ll.value and parts[3] == n
    # ell = -1/2 (sum quad + sum logdet) - n/2 log 2 pi (Alg.5 summed, Q2)
    assert abs(parts[0] - (-0.5 * (parts[1] + parts[2]) - 0.5 * n * math.log(2 * math.pi))) \
        <= 1e-12 * abs(parts[0])
    L.sbv_destroy(h)
    opts = sbv.sbv_opts(3, None, 0)
    h2 = ctypes.c_void_p()
    assert L.sbv_prepare_ex(ctypes.c_void_p(Xd.data_ptr()), n, d, bs, m,
                            sc.ctypes.data_as(ctypes.c_void_p), ctypes.byref(opts), ctypes.byref(h2)) == 0
    ll2 = ctypes.c_double()
    assert L.sbv_loglik(h2, ctypes.c_void_p(yd.data_ptr()), th.ctypes.data_as(ctypes.c_void_p),
                        ctypes.byref(ll2)) == 0
    assert ll2.value == ll.value
    L.sbv_destroy(h2)
    # errors through the ABI: NULL handle out, bad bs
    assert L.sbv_prepare(ctypes.c_void_p(Xd.data_ptr()), n, d, 0, m,
                         sc.ctypes.data_as(ctypes.c_void_p), ctypes.byref(h2)) == 1
    assert not h2.value


@pytest.mark.parametrize("world", [2, 3])
def test_h10_exchange_arithmetic_on_one_gpu(sbv, world):
    """Alg.1 Step 5 without NCCL: every rank's shard computed in
    turn on one device (sbv_set_shard), the per-rank chunk partials
    concatenated in rank order (the allgather layout) and reduced by k_final
    (sbv_reduce_partials): ell and every block term bit-identical to one GPU."""
    import torch
    n, d, bs, m = 60_000, 10, 50, 100
    X = torch.from_numpy(si.make_X(n, d, seed=1)).cuda()
    y = torch.from_numpy(si.make_y(si.make_X(n, d, seed=1), seed=2)).cuda()
    theta = si.default_theta(d, nu=2.5, tau2=1e-4)
    scale = si.default_scale(d)
    h1 = sbv.prepare(X, bs, m, scale)
    ll1 = h1.loglik(y, theta)
    parts1 = h1.loglik_parts(y, theta)
    terms1, _, _ = h1.block_terms(y, theta)
    k = len(terms1)
    partials, merged = [], np.full(k, np.nan)
    hs = []
    for r in range(world):
        h = sbv.Handle(seed=3)
        h.set_shard(r, world)
        h.prepare(X, bs, m, scale)
        partials.append(h.loglik_partials(y, theta))
        tr, _, _ = h.block_terms(y, theta)
        owned = sbv.shard_blocks(k, r, world)
        assert np.isnan(np.delete(tr, owned)).all()
        merged[owned] = tr[owned]
        with pytest.raises(sbv.SBVError) as e:  # no communicator: loglik refuses
            h.loglik(y, theta)
        assert e.value.code == 7
        hs.append(h)
    np.testing.assert_array_equal(merged, terms1)
    allp = np.concatenate(partials)
    for h in hs:
        parts = h.reduce_partials(allp)
        assert parts[0] == ll1, (parts[0], ll1)
        np.testing.assert_array_equal(parts, parts1)


def test_prepare_with_given_partition(sbv, orc):
    """sbv_prepare_blocks: the block partition given (Alg.1 input K):
    layout, centroids and kNN of the given blocks against the oracle's O4-O6 on
    the same partition, then the likelihood."""
    import torch
    n, d, m = 4000, 5, 40
    X = si.make_X(n, d, seed=61)
    y = si.make_y(X, seed=62)
    scale = si.default_scale(d)
    theta = si.default_theta(d, nu=1.5, tau2=1e-4)
    # a partition the GPU path would never produce: grid cells in dims 0-1,
    # block ids shuffled (zeta order = id)
    cell = (np.floor(X[:, 0] * 6) * 6 + np.floor(X[:, 1] * 6)).astype(np.int64)
    ids = np.unique(cell)
    relabel = np.random.default_rng(63).permutation(len(ids))
    bo = relabel[np.searchsorted(ids, cell)].astype(np.int32)
    k = len(ids)
    h = sbv.Handle(seed=3)
    h.prepare_blocks(torch.from_numpy(X).cuda(), torch.from_numpy(bo).cuda(), m, scale, k=k)
    S = orc.scale(X, scale)
    perm_o, off_o = orc.layout(bo, k)
    C_o = orc.centroids(S, perm_o, off_o)
    nbr_o, cnt_o = orc.knn(S, perm_o, off_o, C_o, m)
    bo_g, off_g, perm_g, C_g = h.blocks()
    np.testing.assert_array_equal(bo_g, bo)
    np.testing.assert_array_equal(off_g, off_o)
    np.testing.assert_array_equal(perm_g, perm_o)
    np.testing.assert_array_equal(C_g, C_o)
    nbr, cnt = h.neighbors()
    np.testing.assert_array_equal(cnt, cnt_o)
    np.testing.assert_array_equal(nbr, nbr_o)
    assert (h.anchors() == -1).all()
    P = dict(perm=perm_o, off=off_o, nbr=nbr_o, cnt=cnt_o)
    compare_all("given_partition", h, orc, X, y, torch.from_numpy(y).cuda(), P, theta)
    # host block ids give the same handle state; bad ids are rejected
    h2 = sbv.Handle(seed=3)
    h2.prepare_blocks(X, bo, m, scale, k=k)
    assert h2.loglik(y, theta) == h.loglik(torch.from_numpy(y).cuda(), theta)
    bad = bo.copy()
    bad[5] = k
    with pytest.raises(sbv.SBVError) as e:
        sbv.Handle(seed=3).prepare_blocks(X, bad, m, scale, k=k)
    assert e.value.code == 1
    empty = bo.copy()
    empty[empty == 0] = 1  # block 0 empty
    with pytest.raises(sbv.SBVError) as e:
        sbv.Handle(seed=3).prepare_blocks(X, empty, m, scale, k=k)
    assert e.value.code == 1


def test_bruteforce_knn_m_above_grid_limit(sbv, orc):
    """m > 960 takes the brute-force kNN kernel (prep_kernels.cu): indices and
    terms against the oracle; N_t up to ~1100 in H8."""
    import torch
    n, d, bs, m = 5000, 4, 50, 1000
    X = si.make_X(n, d, seed=71)
    y = si.make_y(X, seed=72)
    scale = np.array([0.2, 0.3, 1.0, 2.0])
    theta = np.array([1.2, 0.2, 0.3, 1.0, 2.0, 2.5, 1e-3])
    h = sbv.prepare(torch.from_numpy(X).cuda(), bs, m, scale)
    P = orc.prepare(X, bs, m, scale, 3)
    nbr, cnt = h.neighbors()
    np.testing.assert_array_equal(cnt, P["cnt"])
    np.testing.assert_array_equal(nbr, P["nbr"])
    assert h.stats()["max_N"] > 1000
    compare_all("knn_bruteforce_m1000", h, orc, X, y, torch.from_numpy(y).cuda(), P, theta)


def test_tau2_zero_informational(sbv, orc):
    """Q19: at tau2 = 0 the per-block conditioning reaches ~1e8 (cfg2 density),
    so parity is informational: the errors are reported, and only loosely gated."""
    import torch
    c = si.CONFIGS["cfg1"]
    n, d, bs, m = c["n"], c["d"], c["bs"], c["m"]
    X = si.make_X(n, d, seed=1)
    y = si.make_y(X, seed=2)
    theta = si.default_theta(d, nu=c["nu"], tau2=0.0)
    h = sbv.prepare(torch.from_numpy(X).cuda(), bs, m, si.default_scale(d))
    P = orc.prepare(X, bs, m, si.default_scale(d), 3)
    ll_o, terms_o, quads_o, logdets_o = orc.loglik(X, y, P["perm"], P["off"], P["nbr"], P["cnt"],
                                                    theta, return_terms=True)
    terms, _, _ = h.block_terms(torch.from_numpy(y).cuda(), theta)
    ll = h.loglik(torch.from_numpy(y).cuda(), theta)
    q18b, strict = term_errors(terms, terms_o, quads_o, logdets_o, np.diff(P["off"]))
    report("tau2_zero_cfg1", max_rel_term_q18b=float(q18b.max()), max_rel_term_strict=float(strict.max()),
           rel_ll=abs(ll - ll_o) / abs(ll_o))
    assert np.isfinite(ll) and abs(ll - ll_o) <= 1e-6 * abs(ll_o)


def test_cfg4_shape_sampled(sbv, orc):
    """BASELINE.json configs[3] shape at n = 5M (bs=100, m=400, nu=3.5, d=10):
    anchors / layout / centroids in full, kNN sets and block terms of sampled
    blocks including the largest N_t and the deepest prefix levels."""
    import torch
    n, d, bs, m, nu = 5_000_000, 10, 100, 400, 3.5
    X = si.make_X(n, d, seed=1)
    y = si.make_y(X, seed=2, kind="iid")
    sc = si.default_scale(d)
    theta = si.default_theta(d, nu=nu, tau2=1e-4)
    h = sbv.prepare(torch.from_numpy(X).cuda(), bs, m, sc)
    k = orc.num_blocks(n, bs)
    np.testing.assert_array_equal(h.anchors(), orc.anchors(n, k, 3))
    S = orc.scale(X, sc)
    bo, off, perm, C = h.blocks()
    perm_o, off_o = orc.layout(bo, k)
    np.testing.assert_array_equal(perm, perm_o)
    np.testing.assert_array_equal(off, off_o)
    np.testing.assert_array_equal(C, orc.centroids(S, perm, off))
    rng = np.random.default_rng(8)
    anc = h.anchors()
    smp = np.setdiff1d(rng.choice(n, 2000, replace=False), anc)
    bo_s = orc.rac(np.concatenate([S[anc], S[smp]]), np.arange(k, dtype=np.int32))[k:]
    np.testing.assert_array_equal(bo[smp], bo_s)
    nbr, cnt = h.neighbors()
    sizes = np.diff(off)
    Nt = np.minimum(m, off[:-1]) + sizes
    big = np.argsort(-Nt, kind="stable")[:3]
    ts = np.unique(np.concatenate([[0, 1, k - 1, k - 2], big, rng.choice(k, 4, replace=False)]))
    assert Nt[big[0]] >= 700
    st = h.stats()
    assert st["max_N"] == Nt.max()
    terms, _, _ = h.block_terms(torch.from_numpy(y).cuda(), theta)
    worst = 0.0
    for t in ts:
        ref = orc.knn_block(S, perm, off, C, int(t), m)
        assert cnt[t] == len(ref), t
        np.testing.assert_array_equal(nbr[t, :cnt[t]], ref, err_msg=f"block {t}")
        to, qo, lo = orc.block_term_at(X, y, perm, off, nbr, cnt, int(t), theta)
        b = max(abs(to), 0.5 * (abs(qo) + abs(lo)) + 0.5 * sizes[t] * math.log(2 * math.pi))
        worst = max(worst, abs(terms[t] - to) / b)
        assert abs(terms[t] - to) <= TOL_TERM * b, (t, terms[t], to)
    report("cfg4_shape_5M_sampled", blocks=[int(t) for t in ts], max_N=int(Nt.max()),
           max_rel_term_q18b=worst)


def test_graph_replay_bit_identical(sbv, orc):
    """sbv_set_graph (the cfg1 latency path): the captured H7 -> H8 -> H9 graph
    gives the stream path's ell bit for bit, for a new theta without
    re-capture, a new y buffer, a different nu and after a re-prepare; the
    oracle pins the first value (north-star 1e-9)."""
    import torch
    n, d, bs, m = 20_000, 10, 20, 60  # cfg1 shape
    X = si.make_X(n, d, seed=61)
    y = si.make_y(X, seed=62)
    scale = si.default_scale(d)
    Xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
    thetas = [si.default_theta(d, nu=2.5, tau2=1e-4), si.default_theta(d, nu=2.5, tau2=3e-3)]
    thetas[1][0] = 1.7
    thetas[1][3] *= 1.3
    th_nu = si.default_theta(d, nu=1.5, tau2=1e-4)
    ref = sbv.Handle(seed=3)
    ref.prepare(Xd, bs, m, scale)
    want = [ref.loglik(yd, t) for t in thetas + [th_nu]]
    h = sbv.Handle(seed=3)
    h.set_graph(True)
    h.prepare(Xd, bs, m, scale)
    got = [h.loglik(yd, thetas[0]), h.loglik(yd, thetas[1]), h.loglik(yd, thetas[0]), h.loglik(yd, th_nu)]
    assert got == [want[0], want[1], want[0], want[2]]
    y2 = yd.clone()
    assert h.loglik(y2, thetas[1]) == want[1]
    h.prepare(Xd, bs, m, scale)
    assert h.loglik(y2, thetas[0]) == want[0]
    P = orc.prepare(X, bs, m, scale, 3)
    ll_o = orc.loglik(X, y, P["perm"], P["off"], P["nbr"], P["cnt"], thetas[0])
    report("graph_replay_cfg1", rel_ll=abs(want[0] - ll_o) / abs(ll_o))
    assert abs(want[0] - ll_o) <= TOL_LL * abs(ll_o)


def test_prepare_from_freed_temporary_on_side_stream(sbv):
    """sbv.h: X is read only during the call.  A handle on a non-blocking side
    stream prepares from a temporary device tensor that is freed on return and
    whose memory torch immediately reuses (overwritten with NaN on its own
    stream): ell must equal the default-stream handle's bit for bit."""
    import torch
    n, d, bs, m = 50_000, 10, 50, 100
    X = si.make_X(n, d, seed=71)
    yd = torch.from_numpy(si.make_y(X, seed=72)).cuda()
    scale = si.default_scale(d)
    theta = si.default_theta(d, nu=2.5, tau2=1e-4)
    ref = sbv.Handle(seed=3)
    ref.prepare(torch.from_numpy(X).cuda(), bs, m, scale)
    want = ref.loglik(yd, theta)
    side = torch.cuda.Stream()
    h = sbv.Handle(seed=3, stream=side)
    for _ in range(3):
        Xt = torch.from_numpy(X).cuda()
        h.prepare(Xt, bs, m, scale)
        del Xt
        junk = torch.full((n, d), float("nan"), dtype=torch.float64, device="cuda")  # reuses the block
        del junk
    torch.cuda.synchronize()
    assert h.loglik(yd, theta) == want
