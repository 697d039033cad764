"""Gradient vs central differences of sbv_loglik at cfg2's full size, for several
steps and two kinds of y (diagnoses FD noise ~1/h vs a systematic difference)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import sbv_inputs as si
import paper_2504_12004_b200 as sbv
c = si.CONFIGS["cfg2"]
n, d, bs, m = c["n"], c["d"], c["bs"], c["m"]
Xh = si.make_X(n, d, seed=1)
X = torch.from_numpy(Xh).cuda()
theta = si.default_theta(d, nu=c["nu"], tau2=1e-4)
h = sbv.Handle(seed=3)
h.prepare(X, bs, m, si.default_scale(d))
idx = [0, *range(1, d + 1), d + 2]
for kind in ("smooth", "iid"):
    y = torch.from_numpy(si.make_y(Xh, seed=2, kind=kind)).cuda()
    ll, g = h.loglik_grad(y, theta)
    base = np.maximum(np.abs(g), np.abs(h.block_grads()).sum(0))
    for step in (1e-6, 1e-5, 1e-4, 1e-3):
        fd = np.zeros(len(idx))
        for k, i in enumerate(idx):
            def D(s):
                tp, tm = theta.copy(), theta.copy()
                tp[i] += s * theta[i]; tm[i] -= s * theta[i]
                return (h.loglik(y, tp) - h.loglik(y, tm)) / (tp[i] - tm[i])
            fd[k] = (4 * D(step) - D(2 * step)) / 3
        rel = np.abs(g - fd) / base
        print(json.dumps({"y": kind, "step": step, "max_rel": float(rel.max()),
                          "rel": [float("%.2e" % v) for v in rel]}))
