"""torchrun check: ell from N ranks (blocks sharded, NCCL) == ell from 1 GPU, bitwise;
per-block terms of all ranks merge into the single-GPU terms.  Prints MGPU_OK."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2504_12004_b200 as sbv  # noqa: E402
import sbv_inputs as si  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    n, d, bs, m = int(os.environ.get("MGPU_N", "60000")), 10, 50, 100
    X = si.make_X(n, d, seed=1)
    y = si.make_y(X, seed=2)
    theta = si.default_theta(d, nu=2.5, tau2=1e-4)
    scale = si.default_scale(d)
    obj = [sbv.comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    h = sbv.Handle(seed=3)
    h.comm_init(obj[0], rank, world)
    h.prepare(torch.from_numpy(X).to(dev), bs, m, scale)
    ll_w = h.loglik(torch.from_numpy(y).to(dev), theta)
    terms_w, _, _ = h.block_terms(torch.from_numpy(y).to(dev), theta)
    nbr_w, cnt_w = h.neighbors()
    all_terms = [None] * world
    dist.all_gather_object(all_terms, terms_w)
    all_nbr = [None] * world
    dist.all_gather_object(all_nbr, (nbr_w, cnt_w))
    ok = True
    if rank == 0:
        h1 = sbv.Handle(seed=3)  # single-GPU reference on this rank's device
        h1.prepare(torch.from_numpy(X).to(dev), bs, m, scale)
        ll_1 = h1.loglik(torch.from_numpy(y).to(dev), theta)
        terms_1, _, _ = h1.block_terms(torch.from_numpy(y).to(dev), theta)
        nbr_1, cnt_1 = h1.neighbors()
        merged = np.full_like(terms_1, np.nan)
        mn = np.full_like(nbr_1, -2)
        mc = np.full_like(cnt_1, -2)
        for r in range(world):
            owned = sbv.shard_blocks(len(terms_1), r, world)
            merged[owned] = all_terms[r][owned]
            mn[owned] = all_nbr[r][0][owned]
            mc[owned] = all_nbr[r][1][owned]
        checks = {"ll": ll_w == ll_1, "terms": bool(np.array_equal(merged, terms_1)),
                  "nbr": bool(np.array_equal(mn, nbr_1)), "cnt": bool(np.array_equal(mc, cnt_1))}
        print(f"ll world={world}: {ll_w!r}  ll 1-GPU: {ll_1!r}  checks: {checks}")
        if not checks["terms"]:
            bad = np.where(merged != terms_1)[0]
            print("terms differ at", bad[:10], merged[bad[:5]], terms_1[bad[:5]])
        if not checks["nbr"]:
            bad = np.where((mn != nbr_1).any(1))[0]
            print("nbr differ at", bad[:10], mn[bad[0]][:8], nbr_1[bad[0]][:8])
        ok = all(checks.values())
        print("MGPU_OK" if ok else "MGPU_FAIL")
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
