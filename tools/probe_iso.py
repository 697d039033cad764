"""Prepare stage times at n=2M, d=10 for the paper's anisotropic scaling vs an
isotropic one (grid pruning over <= 3 dims is weak when all 10 dims matter)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import sbv_inputs as si
import paper_2504_12004_b200 as sbv
n, d = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000, 10
X = torch.from_numpy(si.make_X(n, d, seed=1)).cuda()
for name, sc in [("aniso", si.default_scale(d)), ("iso0.5", np.full(d, 0.5))]:
    h = sbv.Handle(seed=3, profile=True)
    for _ in range(2):
        h.prepare(X, 100, 200, sc)
    print(json.dumps({"scale": name, "grid": os.environ.get("SBV_GRID", "1"),
                      "prep": {k: round(v, 2) for k, v in h.stage_times(True).items()}}))
