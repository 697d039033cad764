"""Gradient stage probe (cfg shape): sbv_loglik_grad stage times via the library's CUDA events."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import sbv_inputs as si
import paper_2504_12004_b200 as sbv
name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
c = dict(si.CONFIGS[name])
if len(sys.argv) > 2: c["n"] = int(sys.argv[2])
X = torch.from_numpy(si.make_X(c["n"], c["d"], seed=1)).cuda()
y = torch.randn(c["n"], dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(2))
theta = si.default_theta(c["d"], nu=c["nu"], tau2=1e-4)
h = sbv.Handle(seed=3, profile=True)
h.prepare(X, c["bs"], c["m"], si.default_scale(c["d"]))
for r in range(3):
    ll, g = h.loglik_grad(y, theta)
    print(json.dumps({"rep": r, "ll": ll, "grad0": float(g[0]), "stages": h.stage_times(False)}))
h.loglik(y, theta)
print(json.dumps({"loglik_stages": h.stage_times(False)}))
