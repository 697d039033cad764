"""Multi-process paths.

CPU (gloo, world_size 2): the block shard of every rank (sbv_shard_blocks, the
same host function sbv_prepare_h uses) partitions the blocks exactly, follows
the 64-block round-robin chunk rule, and balances the kNN cost (prefix length).

GPU (>= 2 devices, torchrun): the log-likelihood from 2 ranks (blocks sharded,
NCCL allgather of chunk partials) is bit-identical to the 1-GPU value, and the
per-block terms of both ranks merge into the 1-GPU terms.
"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _shard_worker(rank, world, port, bc, out):
    sys.path.insert(0, ROOT)
    from paper_2504_12004_b200 import build
    import paper_2504_12004_b200 as sbv
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    mine = sbv.shard_blocks(bc, rank, world).tolist()
    gathered = [None] * world
    dist.all_gather_object(gathered, mine)
    if rank == 0:
        out.put(gathered)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("bc", [1, 65, 10_000])
def test_block_shards_partition_and_balance_gloo(bc):
    from paper_2504_12004_b200 import build
    build.build()
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, bc, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    allb = sorted(b for g in gathered for b in g)
    assert allb == list(range(bc))  # exact partition
    for r, g in enumerate(gathered):
        assert g == sorted(g)
        for b in g:
            assert (b // 64) % world == r  # 64-block chunks dealt round-robin
    if bc >= 1000:  # kNN cost of block t ~ its zeta prefix ~ t: balanced within 5%
        costs = [sum(g) for g in gathered]
        assert max(costs) / min(costs) < 1.05


@pytest.mark.gpu
def test_two_gpu_loglik_bit_identical():
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tools", "mgpu_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "MGPU_OK" in r.stdout
