"""Thin ctypes binding of libsbv (include/sbv.h): argument marshalling only.

Every step of the path runs in the CUDA library; this module converts numpy
arrays / torch tensors (host or device) to pointers and C status codes to
exceptions.  There is no CPU fallback: if libsbv.so is missing or no CUDA
device is present the calls raise.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SBV_LIB") or os.path.join(HERE, "libsbv.so")

SBV_OK, SBV_ERR_ARG, SBV_ERR_CUDA, SBV_ERR_OOM, SBV_ERR_NOT_PD, SBV_ERR_UNSUPPORTED, \
    SBV_ERR_COMM, SBV_ERR_STATE = range(8)
_NAMES = {0: "OK", 1: "ERR_ARG", 2: "ERR_CUDA", 3: "ERR_OOM", 4: "ERR_NOT_PD",
          5: "ERR_UNSUPPORTED", 6: "ERR_COMM", 7: "ERR_STATE"}

_p = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64


class sbv_opts(ctypes.Structure):
    _fields_ = [("seed", ctypes.c_uint64), ("stream", ctypes.c_void_p), ("profile", ctypes.c_int32)]


class SBVError(RuntimeError):
    def __init__(self, code, msg="", block=-1, stage=0):
        super().__init__(f"libsbv {_NAMES.get(code, code)}: {msg}"
                         + (f" (block {block}, stage {stage})" if block >= 0 else ""))
        self.code, self.block, self.stage = code, block, stage


_lib = None

EXPORTS = ["sbv_abi_version", "sbv_create", "sbv_destroy", "sbv_comm_unique_id", "sbv_comm_init",
           "sbv_shard_blocks",
           "sbv_prepare_h", "sbv_prepare_ex", "sbv_prepare", "sbv_prepare_blocks", "sbv_loglik",
           "sbv_loglik_parts",
           "sbv_block_terms", "sbv_num_blocks", "sbv_get_anchors", "sbv_get_blocks",
           "sbv_get_neighbors", "sbv_stats", "sbv_stage_times", "sbv_last_error",
           "sbv_predict", "sbv_get_prediction", "sbv_simulate", "sbv_set_shard",
           "sbv_partials_size", "sbv_loglik_partials", "sbv_reduce_partials",
           "sbv_loglik_grad", "sbv_set_graph", "sbv_block_grads"]


def lib():
    """Load libsbv.so (never builds implicitly; see paper_2504_12004_b200.build)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise SBVError(SBV_ERR_CUDA, f"{LIB_PATH} not built: run python -m paper_2504_12004_b200.build")
        L = ctypes.CDLL(LIB_PATH)
        L.sbv_abi_version.restype = ctypes.c_int
        L.sbv_create.argtypes = [ctypes.POINTER(sbv_opts), ctypes.POINTER(_p)]
        L.sbv_destroy.argtypes = [_p]
        L.sbv_destroy.restype = None
        L.sbv_comm_unique_id.argtypes = [_p]
        L.sbv_comm_init.argtypes = [_p, _p, _i32, _i32]
        L.sbv_shard_blocks.argtypes = [_i64, _i32, _i32, _p, ctypes.POINTER(_i64)]
        L.sbv_prepare_h.argtypes = [_p, _p, _i64, _i32, _i32, _i32, _p]
        L.sbv_prepare_ex.argtypes = [_p, _i64, _i32, _i32, _i32, _p, ctypes.POINTER(sbv_opts),
                                     ctypes.POINTER(_p)]
        L.sbv_prepare.argtypes = [_p, _i64, _i32, _i32, _i32, _p, ctypes.POINTER(_p)]
        L.sbv_set_shard.argtypes = [_p, _i32, _i32]
        L.sbv_set_graph.argtypes = [_p, _i32]
        L.sbv_block_grads.argtypes = [_p, _p]
        L.sbv_loglik_grad.argtypes = [_p, _p, _p, ctypes.POINTER(ctypes.c_double), _p]
        L.sbv_partials_size.argtypes = [_p, ctypes.POINTER(_i64)]
        L.sbv_loglik_partials.argtypes = [_p, _p, _p, _p]
        L.sbv_reduce_partials.argtypes = [_p, _p, _p]
        L.sbv_prepare_blocks.argtypes = [_p, _p, _i64, _i32, _i64, _p, _i32, _p]
        L.sbv_loglik.argtypes = [_p, _p, _p, ctypes.POINTER(ctypes.c_double)]
        L.sbv_loglik_parts.argtypes = [_p, _p, _p, _p]
        L.sbv_block_terms.argtypes = [_p, _p, _p, _p, _p, _p]
        L.sbv_num_blocks.argtypes = [_p, ctypes.POINTER(_i64)]
        L.sbv_get_anchors.argtypes = [_p, _p]
        L.sbv_get_blocks.argtypes = [_p, _p, _p, _p, _p]
        L.sbv_get_neighbors.argtypes = [_p, _p, _p]
        L.sbv_stats.argtypes = [_p, _p]
        L.sbv_stage_times.argtypes = [_p, _i32, _p, _p, _i32, ctypes.POINTER(_i32)]
        L.sbv_last_error.argtypes = [_p, ctypes.POINTER(_i64), ctypes.POINTER(_i32),
                                     ctypes.POINTER(ctypes.c_char_p)]
        L.sbv_predict.argtypes = [_p, _p, _i64, _i32, _i32, _p, _p, _p, _p]
        L.sbv_get_prediction.argtypes = [_p, ctypes.POINTER(_i64), _p, _p, _p, _p, _p, _p]
        L.sbv_simulate.argtypes = [_p, _p, _p, _i64, _i32, ctypes.c_uint64, ctypes.c_double,
                                   _p, _p, _p, _p]
        _lib = L
    return _lib


def _ptr(a):
    """(pointer, keepalive) for a numpy array or torch tensor (host or device)."""
    if a is None:
        return None, None
    if hasattr(a, "data_ptr"):  # torch tensor
        if not a.is_contiguous():
            raise SBVError(SBV_ERR_ARG, "tensor must be contiguous")
        return _p(a.data_ptr()), a
    arr = np.ascontiguousarray(a)
    return _p(arr.ctypes.data), arr


def _f64(a):
    if hasattr(a, "data_ptr"):
        import torch
        if a.dtype != torch.float64:
            raise SBVError(SBV_ERR_ARG, "expected float64 tensor")
        return a.contiguous()
    return np.ascontiguousarray(a, dtype=np.float64)


def shard_blocks(bc: int, rank: int, world: int):
    """Zeta ids of the blocks owned by `rank` (host-only; sbv_shard_blocks)."""
    cnt = _i64(0)
    rc = lib().sbv_shard_blocks(bc, rank, world, None, ctypes.byref(cnt))
    if rc:
        raise SBVError(rc, "sbv_shard_blocks")
    out = np.empty(max(cnt.value, 1), dtype=np.int32)
    lib().sbv_shard_blocks(bc, rank, world, out.ctypes.data_as(_p), ctypes.byref(cnt))
    return out[:cnt.value].copy()


def comm_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    rc = lib().sbv_comm_unique_id(buf)
    if rc:
        raise SBVError(rc, "ncclGetUniqueId failed")
    return buf.raw


class Handle:
    """An sbv_handle: prepared state of Alg.1 Steps 1-3 living on one GPU."""

    def __init__(self, seed: int = 3, stream=None, profile: bool = False):
        L = lib()
        self._h = _p()
        st = 0
        if stream is not None:
            st = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        self._opts = sbv_opts(seed, _p(st) if st else None, 1 if profile else 0)
        rc = L.sbv_create(ctypes.byref(self._opts), ctypes.byref(self._h))
        if rc:
            raise SBVError(rc, "sbv_create failed (no CUDA device?)")
        self.n = self.d = self.bs = self.m = 0

    # -- errors
    def last_error(self):
        b, s, msg = _i64(0), _i32(0), ctypes.c_char_p()
        lib().sbv_last_error(self._h, ctypes.byref(b), ctypes.byref(s), ctypes.byref(msg))
        return b.value, s.value, (msg.value or b"").decode()

    def _check(self, rc):
        if rc:
            b, s, msg = self.last_error()
            raise SBVError(rc, msg, b if rc == SBV_ERR_NOT_PD else -1, s)

    # -- lifecycle
    def comm_init(self, unique_id: bytes, rank: int, world: int):
        buf = ctypes.create_string_buffer(unique_id, 128)
        self._check(lib().sbv_comm_init(self._h, buf, rank, world))

    def set_graph(self, enable: bool = True):
        """sbv_set_graph: replay loglik from a CUDA graph (device y, one GPU)."""
        self._check(lib().sbv_set_graph(self._h, 1 if enable else 0))

    def set_shard(self, rank: int, world: int):
        """sbv_set_shard: shard without a communicator (caller-side exchange)."""
        self._check(lib().sbv_set_shard(self._h, rank, world))

    def loglik_partials(self, y, theta):
        y = _f64(y)
        th = np.ascontiguousarray(theta, dtype=np.float64)
        py, _k = _ptr(y)
        cnt = _i64(0)
        rc = lib().sbv_partials_size(self._h, ctypes.byref(cnt))
        self._check(rc)
        out = np.zeros(cnt.value)
        self._check(lib().sbv_loglik_partials(self._h, py, th.ctypes.data_as(_p), out.ctypes.data_as(_p)))
        return out

    def reduce_partials(self, all_partials):
        a = np.ascontiguousarray(all_partials, dtype=np.float64)
        parts = np.zeros(4)
        self._check(lib().sbv_reduce_partials(self._h, a.ctypes.data_as(_p), parts.ctypes.data_as(_p)))
        return parts

    def prepare(self, X, bs: int, m: int, scale):
        X = _f64(X)
        n, d = X.shape
        sc = np.ascontiguousarray(scale, dtype=np.float64)
        if sc.shape != (d,):
            raise SBVError(SBV_ERR_ARG, "scale must have length d")
        px, _k = _ptr(X)
        self._check(lib().sbv_prepare_h(self._h, px, n, d, bs, m, sc.ctypes.data_as(_p)))
        self.n, self.d, self.bs, self.m = n, d, bs, m
        return self

    def prepare_blocks(self, X, block_of, m: int, scale, k: int = None):
        """sbv_prepare_blocks: the block partition is given (block id = zeta position)."""
        X = _f64(X)
        n, d = X.shape
        sc = np.ascontiguousarray(scale, dtype=np.float64)
        if sc.shape != (d,):
            raise SBVError(SBV_ERR_ARG, "scale must have length d")
        if hasattr(block_of, "data_ptr"):
            bo = block_of.contiguous()
            pb = bo.data_ptr()
            kk = int(bo.max().item()) + 1 if k is None else k
        else:
            bo = np.ascontiguousarray(block_of, dtype=np.int32)
            pb = bo.ctypes.data
            kk = int(bo.max()) + 1 if k is None else k
        px, _k = _ptr(X)
        self._check(lib().sbv_prepare_blocks(self._h, px, n, d, kk, _p(pb), m, sc.ctypes.data_as(_p)))
        self.n, self.d, self.bs, self.m = n, d, max(1, n // kk), m
        return self

    def destroy(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().sbv_destroy(self._h)
            self._h = _p()

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass

    # -- Steps 4-5
    def loglik(self, y, theta) -> float:
        y = _f64(y)
        th = np.ascontiguousarray(theta, dtype=np.float64)
        py, _k = _ptr(y)
        out = ctypes.c_double(0.0)
        self._check(lib().sbv_loglik(self._h, py, th.ctypes.data_as(_p), ctypes.byref(out)))
        return out.value

    def loglik_grad(self, y, theta):
        """(ell, d ell / d (sigma2, beta_1..beta_d, tau2)) -- sbv_loglik_grad."""
        y = _f64(y)
        th = np.ascontiguousarray(theta, dtype=np.float64)
        py, _k = _ptr(y)
        out = ctypes.c_double(0.0)
        g = np.zeros(self.d + 2)
        self._check(lib().sbv_loglik_grad(self._h, py, th.ctypes.data_as(_p), ctypes.byref(out),
                                          g.ctypes.data_as(_p)))
        return out.value, g

    def block_grads(self):
        """sbv_block_grads: per-block gradients of the last loglik_grad, (bc, d+2)."""
        out = np.zeros((self.num_blocks(), self.d + 2))
        self._check(lib().sbv_block_grads(self._h, out.ctypes.data_as(_p)))
        return out

    def loglik_parts(self, y, theta):
        y = _f64(y)
        th = np.ascontiguousarray(theta, dtype=np.float64)
        py, _k = _ptr(y)
        parts = np.zeros(4)
        self._check(lib().sbv_loglik_parts(self._h, py, th.ctypes.data_as(_p),
                                           parts.ctypes.data_as(_p)))
        return parts

    def block_terms(self, y, theta, raise_not_pd: bool = False):
        y = _f64(y)
        th = np.ascontiguousarray(theta, dtype=np.float64)
        py, _k = _ptr(y)
        k = self.num_blocks()
        terms, quad, logdet = np.empty(k), np.empty(k), np.empty(k)
        rc = lib().sbv_block_terms(self._h, py, th.ctypes.data_as(_p), terms.ctypes.data_as(_p),
                                   quad.ctypes.data_as(_p), logdet.ctypes.data_as(_p))
        if rc and (rc != SBV_ERR_NOT_PD or raise_not_pd):
            self._check(rc)
        return terms, quad, logdet

    # -- introspection
    def num_blocks(self) -> int:
        k = _i64(0)
        self._check(lib().sbv_num_blocks(self._h, ctypes.byref(k)))
        return k.value

    def anchors(self):
        a = np.empty(self.num_blocks(), dtype=np.int32)
        self._check(lib().sbv_get_anchors(self._h, a.ctypes.data_as(_p)))
        return a

    def blocks(self):
        k = self.num_blocks()
        bo = np.empty(self.n, dtype=np.int32)
        off = np.empty(k + 1, dtype=np.int64)
        perm = np.empty(self.n, dtype=np.int32)
        C = np.empty((k, self.d), dtype=np.float64)
        self._check(lib().sbv_get_blocks(self._h, bo.ctypes.data_as(_p), off.ctypes.data_as(_p),
                                         perm.ctypes.data_as(_p), C.ctypes.data_as(_p)))
        return bo, off, perm, C

    # -- prediction
    def predict(self, X_star, bs_pred: int, m_pred: int, y, theta):
        """Conditional mean and variance at X_star (Eq.3 / Sec.4.1 per test block).
        Outputs are numpy arrays unless X_star is a CUDA tensor (then tensors)."""
        Xs = _f64(X_star)
        y = _f64(y)
        th = np.ascontiguousarray(theta, dtype=np.float64)
        ns = Xs.shape[0]
        if hasattr(Xs, "data_ptr") and Xs.is_cuda:
            import torch
            mean = torch.empty(ns, dtype=torch.float64, device=Xs.device)
            var = torch.empty(ns, dtype=torch.float64, device=Xs.device)
        else:
            mean, var = np.empty(ns), np.empty(ns)
        px, _k1 = _ptr(Xs)
        py, _k2 = _ptr(y)
        pm, _k3 = _ptr(mean)
        pv, _k4 = _ptr(var)
        self._check(lib().sbv_predict(self._h, px, ns, bs_pred, m_pred, py, th.ctypes.data_as(_p), pm, pv))
        self._last_pred = (ns, m_pred)
        return mean, var

    def prediction_structure(self):
        """(anchors, block_of, off, perm, nbr (original training indices), cnt) of the last predict."""
        ks = _i64(0)
        self._check(lib().sbv_get_prediction(self._h, ctypes.byref(ks), None, None, None, None, None, None))
        k = ks.value
        ns, mp = self._last_pred
        anc = np.empty(k, np.int32)
        bo = np.empty(ns, np.int32)
        off = np.empty(k + 1, np.int64)
        perm = np.empty(ns, np.int32)
        nbr = np.empty((k, max(mp, 1)), np.int32)
        cnt = np.empty(k, np.int32)
        self._check(lib().sbv_get_prediction(self._h, ctypes.byref(ks), *[a.ctypes.data_as(_p) for a in
                                                                         (anc, bo, off, perm, nbr, cnt)]))
        return anc, bo, off, perm, nbr[:, :mp], cnt

    def simulate(self, mean, var, n_sim: int, seed: int, ci_level: float = 0.95):
        """Sec.5.5 conditional simulation: (sample mean, sample sd, ci_lo, ci_hi)."""
        m = np.ascontiguousarray(mean.cpu().numpy() if hasattr(mean, "cpu") else mean, dtype=np.float64)
        v = np.ascontiguousarray(var.cpu().numpy() if hasattr(var, "cpu") else var, dtype=np.float64)
        outs = [np.empty(m.shape[0]) for _ in range(4)]
        self._check(lib().sbv_simulate(self._h, m.ctypes.data_as(_p), v.ctypes.data_as(_p), m.shape[0],
                                       n_sim, seed, ci_level, *[o.ctypes.data_as(_p) for o in outs]))
        return tuple(outs)

    def neighbors(self):
        k = self.num_blocks()
        m = self.m
        nbr = np.empty((k, max(m, 1)), dtype=np.int32)
        cnt = np.empty(k, dtype=np.int32)
        self._check(lib().sbv_get_neighbors(self._h, nbr.ctypes.data_as(_p), cnt.ctypes.data_as(_p)))
        return (nbr[:, :m] if m > 0 else np.empty((k, 0), np.int32)), cnt

    def stats(self) -> dict:
        s = np.zeros(9)
        self._check(lib().sbv_stats(self._h, s.ctypes.data_as(_p)))
        keys = ["flops", "entries", "max_N", "min_bs", "max_bs", "k_local", "knn_pairs",
                "rac_pairs", "h8_bytes"]
        return dict(zip(keys, s.tolist()))

    def stage_times(self, prep: bool = False) -> dict:
        cap = 16
        ms = np.zeros(cap)
        names = (ctypes.c_char_p * cap)()
        cnt = _i32(0)
        self._check(lib().sbv_stage_times(self._h, 1 if prep else 0, ms.ctypes.data_as(_p),
                                          ctypes.cast(names, _p), cap, ctypes.byref(cnt)))
        return {names[i].decode(): float(ms[i]) for i in range(cnt.value)}


def prepare(X, bs: int, m: int, scale, seed: int = 3, stream=None, profile: bool = False,
            comm=None) -> Handle:
    """sbv_prepare(X, n, d, bs, m, scale) -> Handle.  comm = (unique_id, rank, world)."""
    h = Handle(seed=seed, stream=stream, profile=profile)
    if comm is not None:
        h.comm_init(*comm)
    return h.prepare(X, bs, m, scale)
