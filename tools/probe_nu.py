"""H8 time at cfg2 for several smoothness values (general-nu K_nu path vs closed forms)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import sbv_inputs as si
import paper_2504_12004_b200 as sbv
c = si.CONFIGS["cfg2"]
X = torch.from_numpy(si.make_X(c["n"], c["d"], seed=1)).cuda()
y = torch.randn(c["n"], dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(2))
h = sbv.Handle(seed=3, profile=True)
h.prepare(X, c["bs"], c["m"], si.default_scale(c["d"]))
for nu in [2.5, 2.0, 1.0, 0.3, 4.25]:
    th = si.default_theta(c["d"], nu=nu, tau2=1e-4)
    h.loglik(y, th)
    h.loglik(y, th)
    print(json.dumps({"nu": nu, "H8_ms": h.stage_times(False)["H8_block_llh"]}))
