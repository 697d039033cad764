"""Plain FP64 CPU oracle for the Scaled Block Vecchia hot path (arXiv 2504.12004).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  It shares no code with ``paper_2504_12004_b200`` (the CUDA product
path) and neither imports the other.

The arithmetic lives in ``sbv_oracle.c`` (one function per algorithm step, each
citing the PAPER.md passage it follows); this module only loads the shared
library (building it with gcc when missing) and marshals numpy arrays.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sbv_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_u64 = ctypes.c_uint64
_dbl = ctypes.c_double
_p = ctypes.c_void_p


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (-O2 -ffp-contract=off -fopenmp)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fopenmp", "-shared", "-fPIC",
               "-o", _LIB, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        L.orc_scale.argtypes = [_p, _i64, _i32, _p, _p]
        L.orc_splitmix64.argtypes = [_u64, _u64]
        L.orc_splitmix64.restype = _u64
        L.orc_num_blocks.argtypes = [_i64, _i32]
        L.orc_num_blocks.restype = _i64
        L.orc_anchors.argtypes = [_i64, _i64, _u64, _p]
        L.orc_dist2.argtypes = [_p, _p, _i32]
        L.orc_dist2.restype = _dbl
        L.orc_rac.argtypes = [_p, _i64, _i32, _p, _i64, _p]
        L.orc_layout.argtypes = [_p, _i64, _i64, _p, _p]
        L.orc_centroids.argtypes = [_p, _i32, _p, _p, _i64, _p]
        L.orc_knn_block.argtypes = [_p, _i32, _p, _p, _p, _i64, _i32, _p]
        L.orc_knn_block.restype = _i32
        L.orc_knn.argtypes = [_p, _i32, _p, _p, _p, _i64, _i32, _p, _p, _i32]
        L.orc_besselk.argtypes = [_dbl, _dbl]
        L.orc_besselk.restype = _dbl
        L.orc_matern.argtypes = [_dbl, _dbl, _dbl]
        L.orc_matern.restype = _dbl
        L.orc_scaled_distance.argtypes = [_p, _p, _i32, _p]
        L.orc_scaled_distance.restype = _dbl
        L.orc_kernel.argtypes = [_p, _p, _i32, _p, _i32]
        L.orc_kernel.restype = _dbl
        L.orc_block_term.argtypes = [_p, _p, _i32, _p, _i32, _p, _i32, _p, _p, _p, _p, _p]
        L.orc_block_term.restype = ctypes.c_int
        L.orc_loglik.argtypes = [_p, _p, _i64, _i32, _p, _p, _i64, _p, _p, _i32, _p, _i32,
                                 _p, _p, _p, _p, _p, _p]
        L.orc_loglik.restype = ctypes.c_int
        L.orc_block_term_at.argtypes = [_p, _p, _i32, _p, _p, _p, _p, _i32, _i64, _p,
                                        _p, _p, _p, _p]
        L.orc_block_term_at.restype = ctypes.c_int
        L.orc_max_threads.restype = ctypes.c_int
        L.orc_knn_pred.argtypes = [_p, _i64, _i32, _p, _i32, _p]
        L.orc_knn_pred.restype = _i32
        L.orc_predict_block.argtypes = [_p, _p, _p, _i32, _p, _i32, _p, _i32, _p, _p, _p]
        L.orc_predict_block.restype = ctypes.c_int
        L.orc_simulate.argtypes = [_p, _p, _i64, _i32, _u64, _dbl, _p, _p, _p, _p]
        L.orc_kernel_grad.argtypes = [_p, _p, _i32, _p, _i32, _p]
        L.orc_block_grad.argtypes = [_p, _p, _i32, _p, _i32, _p, _i32, _p, _p]
        L.orc_block_grad.restype = ctypes.c_int
        L.orc_loglik_grad.argtypes = [_p, _p, _i32, _p, _p, _i64, _p, _p, _i32, _p, _i32, _p, _p]
        L.orc_loglik_grad.restype = ctypes.c_int
        L.orc_z_crit.argtypes = [_dbl]
        L.orc_z_crit.restype = _dbl
        _lib = L
    return _lib


def _c(a, dtype):
    a = np.ascontiguousarray(a, dtype=dtype)
    return a, a.ctypes.data_as(_p)


def max_threads() -> int:
    return int(lib().orc_max_threads())


# ----------------------------------------------------------------- O1
def scale(X, scale_):
    X, px = _c(X, np.float64)
    s, ps = _c(scale_, np.float64)
    n, d = X.shape
    S = np.empty_like(X)
    lib().orc_scale(px, n, d, ps, S.ctypes.data_as(_p))
    return S


# ----------------------------------------------------------------- O2
def splitmix64(seed: int, i: int) -> int:
    return int(lib().orc_splitmix64(seed, i))


def num_blocks(n: int, bs: int) -> int:
    return int(lib().orc_num_blocks(n, bs))


def anchors(n: int, k: int, seed: int):
    a = np.empty(k, dtype=np.int32)
    lib().orc_anchors(n, k, seed, a.ctypes.data_as(_p))
    return a


# ----------------------------------------------------------------- O3
def dist2(a, b) -> float:
    a, pa = _c(a, np.float64)
    b, pb = _c(b, np.float64)
    return float(lib().orc_dist2(pa, pb, a.shape[0]))


def rac(S, anc):
    S, ps = _c(S, np.float64)
    anc, pa = _c(anc, np.int32)
    n, d = S.shape
    bo = np.empty(n, dtype=np.int32)
    lib().orc_rac(ps, n, d, pa, anc.shape[0], bo.ctypes.data_as(_p))
    return bo


# ----------------------------------------------------------------- O4
def layout(block_of, k: int):
    bo, pb = _c(block_of, np.int32)
    perm = np.empty(bo.shape[0], dtype=np.int32)
    off = np.empty(k + 1, dtype=np.int64)
    lib().orc_layout(pb, bo.shape[0], k, perm.ctypes.data_as(_p), off.ctypes.data_as(_p))
    return perm, off


# ----------------------------------------------------------------- O5
def centroids(S, perm, off):
    S, ps = _c(S, np.float64)
    perm, pp = _c(perm, np.int32)
    off, po = _c(off, np.int64)
    k = off.shape[0] - 1
    C = np.empty((k, S.shape[1]), dtype=np.float64)
    lib().orc_centroids(ps, S.shape[1], pp, po, k, C.ctypes.data_as(_p))
    return C


# ----------------------------------------------------------------- O6
def knn_block(S, perm, off, C, t: int, m: int):
    S, ps = _c(S, np.float64)
    perm, pp = _c(perm, np.int32)
    off, po = _c(off, np.int64)
    C, pc = _c(C, np.float64)
    out = np.empty(max(m, 1), dtype=np.int32)
    c = lib().orc_knn_block(ps, S.shape[1], pp, po, pc, t, m, out.ctypes.data_as(_p))
    return out[:c].copy()


def knn(S, perm, off, C, m: int, nthreads: int = 0):
    S, ps = _c(S, np.float64)
    perm, pp = _c(perm, np.int32)
    off, po = _c(off, np.int64)
    C, pc = _c(C, np.float64)
    k = off.shape[0] - 1
    nbr = np.empty((k, max(m, 1)), dtype=np.int32)
    cnt = np.empty(k, dtype=np.int32)
    lib().orc_knn(ps, S.shape[1], pp, po, pc, k, m, nbr.ctypes.data_as(_p),
                  cnt.ctypes.data_as(_p), nthreads)
    return nbr[:, :m].copy() if m > 0 else np.empty((k, 0), np.int32), cnt


# ----------------------------------------------------------------- O7
def matern(r: float, sigma2: float, nu: float) -> float:
    return float(lib().orc_matern(r, sigma2, nu))


def besselk(nu: float, r: float) -> float:
    return float(lib().orc_besselk(nu, r))


def scaled_distance(xa, xb, beta) -> float:
    xa, pa = _c(xa, np.float64)
    xb, pb = _c(xb, np.float64)
    beta, pbeta = _c(beta, np.float64)
    return float(lib().orc_scaled_distance(pa, pb, xa.shape[0], pbeta))


def kernel(xa, xb, theta, same: bool) -> float:
    xa, pa = _c(xa, np.float64)
    xb, pb = _c(xb, np.float64)
    th, pt = _c(theta, np.float64)
    return float(lib().orc_kernel(pa, pb, xa.shape[0], pt, int(same)))


# ----------------------------------------------------------------- O8/O9
class NotPD(RuntimeError):
    def __init__(self, block, stage):
        super().__init__(f"Cholesky failed: block {block}, stage {stage}")
        self.block, self.stage = block, stage


def block_term(X, y, J, B, theta):
    """One block's Alg.5 term.  Returns (term, quad, logdet)."""
    X, px = _c(X, np.float64)
    y, py = _c(y, np.float64)
    J, pj = _c(np.asarray(J, dtype=np.int32).reshape(-1), np.int32)
    B, pB = _c(np.asarray(B, dtype=np.int32).reshape(-1), np.int32)
    th, pt = _c(theta, np.float64)
    out = np.zeros(3)
    st = ctypes.c_int32(0)
    o = out.ctypes.data
    rc = lib().orc_block_term(px, py, X.shape[1], pj, J.shape[0], pB, B.shape[0], pt,
                              _p(o), _p(o + 8), _p(o + 16), ctypes.byref(st))
    if rc != 0:
        raise NotPD(-1, st.value)
    return float(out[0]), float(out[1]), float(out[2])


def block_term_at(X, y, perm, off, nbr, cnt, t: int, theta):
    X, px = _c(X, np.float64)
    y, py = _c(y, np.float64)
    perm, pp = _c(perm, np.int32)
    off, po = _c(off, np.int64)
    m = nbr.shape[1] if nbr.ndim == 2 else 0
    nbr_, pn = _c(nbr if m > 0 else np.zeros((off.shape[0] - 1, 1), np.int32), np.int32)
    cnt, pc = _c(cnt, np.int32)
    th, pt = _c(theta, np.float64)
    out = np.zeros(3)
    st = ctypes.c_int32(0)
    o = out.ctypes.data
    rc = lib().orc_block_term_at(px, py, X.shape[1], pp, po, pn, pc, max(m, 1), t, pt,
                                 _p(o), _p(o + 8), _p(o + 16), ctypes.byref(st))
    if rc != 0:
        raise NotPD(t, st.value)
    return float(out[0]), float(out[1]), float(out[2])


def loglik(X, y, perm, off, nbr, cnt, theta, nthreads: int = 0, return_terms=False):
    """Alg.1 Steps 4-5.  Returns ell (and per-block terms/quads/logdets)."""
    X, px = _c(X, np.float64)
    y, py = _c(y, np.float64)
    perm, pp = _c(perm, np.int32)
    off, po = _c(off, np.int64)
    k = off.shape[0] - 1
    m = nbr.shape[1] if nbr.ndim == 2 else 0
    nbr_, pn = _c(nbr if m > 0 else np.zeros((k, 1), np.int32), np.int32)
    cnt, pc = _c(cnt, np.int32)
    th, pt = _c(theta, np.float64)
    terms = np.empty(k)
    quads = np.empty(k)
    logdets = np.empty(k)
    out = np.zeros(3)
    fb = ctypes.c_int64(0)
    fs = ctypes.c_int32(0)
    rc = lib().orc_loglik(px, py, X.shape[0], X.shape[1], pp, po, k, pn, pc, max(m, 1), pt,
                          nthreads, terms.ctypes.data_as(_p), quads.ctypes.data_as(_p),
                          logdets.ctypes.data_as(_p), out.ctypes.data_as(_p),
                          ctypes.byref(fb), ctypes.byref(fs))
    if rc != 0:
        raise NotPD(fb.value, fs.value)
    if return_terms:
        return float(out[0]), terms, quads, logdets
    return float(out[0])


def prepare(X, bs: int, m: int, scale_, seed: int, nthreads: int = 0):
    """O1-O6 composed: scale, anchors + zeta, RAC, layout, centroids, kNN."""
    n = X.shape[0]
    S = scale(X, scale_)
    k = num_blocks(n, bs)
    anc = anchors(n, k, seed)
    bo = rac(S, anc)
    perm, off = layout(bo, k)
    C = centroids(S, perm, off)
    nbr, cnt = knn(S, perm, off, C, m, nthreads)
    return dict(S=S, k=k, anchors=anc, block_of=bo, perm=perm, off=off, C=C, nbr=nbr, cnt=cnt)


# ----------------------------------------------------------------- O10-O12 (NEXT N2)
def knn_pred(S, c, m: int):
    """Prediction-mode m-NN of centroid c over ALL training rows of S (original indices)."""
    S, ps = _c(S, np.float64)
    c, pc = _c(c, np.float64)
    out = np.empty(max(m, 1), dtype=np.int32)
    k = lib().orc_knn_pred(ps, S.shape[0], S.shape[1], pc, m, out.ctypes.data_as(_p))
    return out[:k].copy()


def predict_block(Xtr, y, Xte, J, B, theta):
    """One test block: (mean, var) of Sec.4.1 restricted to NN(B*)."""
    Xtr, px = _c(Xtr, np.float64)
    y, py = _c(y, np.float64)
    Xte, pt = _c(Xte, np.float64)
    J, pj = _c(np.asarray(J, dtype=np.int32).reshape(-1), np.int32)
    B, pb = _c(np.asarray(B, dtype=np.int32).reshape(-1), np.int32)
    th, pth = _c(theta, np.float64)
    mean = np.empty(B.shape[0])
    var = np.empty(B.shape[0])
    rc = lib().orc_predict_block(px, py, pt, Xtr.shape[1], pj, J.shape[0], pb, B.shape[0], pth,
                                 mean.ctypes.data_as(_p), var.ctypes.data_as(_p))
    if rc != 0:
        raise NotPD(-1, 1)
    return mean, var


def predict(Xtr, y, Xte, bs_pred: int, m_pred: int, scale_, theta, seed: int = 3):
    """Eq.3 prediction: test blocks by the same anchors + RAC (O2-O5) on the
    scaled test inputs, prediction-mode NN over the training set, per-block
    conditional mean / variance.  Returns (mean, var, blocks) in test order."""
    S = scale(Xtr, scale_)
    St = scale(Xte, scale_)
    nt = Xte.shape[0]
    k = num_blocks(nt, bs_pred)
    anc = anchors(nt, k, seed)
    bo = rac(St, anc)
    perm, off = layout(bo, k)
    C = centroids(St, perm, off)
    mean = np.empty(nt)
    var = np.empty(nt)
    nbrs = []
    for t in range(k):
        J = knn_pred(S, C[t], m_pred)
        B = perm[off[t]:off[t + 1]]
        mu, v = predict_block(Xtr, y, Xte, J, B, theta)
        mean[B] = mu
        var[B] = v
        nbrs.append(J)
    return mean, var, dict(anchors=anc, block_of=bo, perm=perm, off=off, C=C, nbr=nbrs)


# ----------------------------------------------------------------- O13 (NEXT N3)
def kernel_grad(xa, xb, theta, same: bool):
    """d K(xa, xb) / d (sigma2, beta_1..beta_d, tau2)."""
    xa, pa = _c(xa, np.float64)
    xb, pb = _c(xb, np.float64)
    th, pt = _c(theta, np.float64)
    out = np.empty(xa.shape[0] + 2)
    lib().orc_kernel_grad(pa, pb, xa.shape[0], pt, int(same), out.ctypes.data_as(_p))
    return out


def block_grad(X, y, J, B, theta):
    """d ell_t / d (sigma2, beta, tau2) of one block (Alg.5 term, nu fixed)."""
    X, px = _c(X, np.float64)
    y, py = _c(y, np.float64)
    J, pj = _c(np.asarray(J, dtype=np.int32).reshape(-1), np.int32)
    B, pB = _c(np.asarray(B, dtype=np.int32).reshape(-1), np.int32)
    th, pt = _c(theta, np.float64)
    g = np.empty(X.shape[1] + 2)
    rc = lib().orc_block_grad(px, py, X.shape[1], pj, J.shape[0], pB, B.shape[0], pt, g.ctypes.data_as(_p))
    if rc == 4:
        raise NotPD(-1, 0)
    if rc != 0:
        raise ValueError("gradient needs a half-integer nu")
    return g


def loglik_grad(X, y, perm, off, nbr, cnt, theta, nthreads: int = 0, return_blocks=False):
    """sum over blocks of d ell_t / d (sigma2, beta, tau2)."""
    X, px = _c(X, np.float64)
    y, py = _c(y, np.float64)
    perm, pp = _c(perm, np.int32)
    off, po = _c(off, np.int64)
    k = off.shape[0] - 1
    m = nbr.shape[1] if nbr.ndim == 2 else 0
    nbr_, pn = _c(nbr if m > 0 else np.zeros((k, 1), np.int32), np.int32)
    cnt, pc = _c(cnt, np.int32)
    th, pt = _c(theta, np.float64)
    P = X.shape[1] + 2
    g = np.empty(P)
    gb = np.empty((k, P))
    rc = lib().orc_loglik_grad(px, py, X.shape[1], pp, po, k, pn, pc, max(m, 1), pt, nthreads,
                               g.ctypes.data_as(_p), gb.ctypes.data_as(_p))
    if rc == 4:
        raise NotPD(-1, 0)
    if rc != 0:
        raise ValueError("gradient needs a half-integer nu")
    return (g, gb) if return_blocks else g


def z_crit(ci_level: float) -> float:
    return float(lib().orc_z_crit(ci_level))


def simulate(mean, var, n_sim: int, seed: int, ci_level: float = 0.95):
    mean, pm = _c(mean, np.float64)
    var, pv = _c(var, np.float64)
    n = mean.shape[0]
    out = [np.empty(n) for _ in range(4)]
    lib().orc_simulate(pm, pv, n, n_sim, seed, z_crit(ci_level), *[o.ctypes.data_as(_p) for o in out])
    return tuple(out)
