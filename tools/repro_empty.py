"""Repro of the given-partition error paths (debug tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SBV_DEBUG"] = "1"
import faulthandler; faulthandler.enable()
import numpy as np, torch
import sbv_inputs as si
import paper_2504_12004_b200 as sbv
n, d, m = 4000, 5, 40
X = si.make_X(n, d, seed=61)
scale = si.default_scale(d)
cell = (np.floor(X[:, 0] * 6) * 6 + np.floor(X[:, 1] * 6)).astype(np.int64)
ids = np.unique(cell)
bo = np.searchsorted(ids, cell).astype(np.int32)
k = len(ids)
for case in ["ok", "bad", "empty"]:
    b = bo.copy()
    if case == "bad": b[5] = k
    if case == "empty": b[b == 0] = 1
    print("case", case, flush=True)
    try:
        h = sbv.Handle(seed=3)
        h.prepare_blocks(X, b, m, scale, k=k)
        print("ok", h.num_blocks(), flush=True)
    except sbv.SBVError as e:
        print("error", e, flush=True)
    del h
print("done", flush=True)
