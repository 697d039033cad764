"""B200 (sm_100a) implementation of the Scaled Block Vecchia log-likelihood
hot path (arXiv 2504.12004) behind the C ABI of include/sbv.h.

    from paper_2504_12004_b200 import prepare
    h = prepare(X, bs=100, m=200, scale=beta)   # Alg.1 Steps 1-3 on the GPU
    ll = h.loglik(y, theta)                     # Alg.1 Steps 4-5 (Alg.5) on the GPU
"""
from .sbv import SBVError, Handle, comm_unique_id, lib, prepare, sbv_opts, shard_blocks  # noqa: F401
