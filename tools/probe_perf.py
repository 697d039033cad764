"""Quick stage-time probe (not the bench): prepare + loglik stage times via the
library's own CUDA events, for a named config.  Usage: python tools/probe_perf.py cfg2 [reps]"""
import json, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import sbv_inputs as si
import paper_2504_12004_b200 as sbv
name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
c = dict(si.CONFIGS[name])
if len(sys.argv) > 3: c["n"] = int(sys.argv[3])
X = torch.from_numpy(si.make_X(c["n"], c["d"], seed=1)).cuda()
y = torch.from_numpy(si.make_y(si.make_X(1000, c["d"], seed=9), seed=2, kind="iid")).cuda()
y = torch.randn(c["n"], dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(2))
theta = si.default_theta(c["d"], nu=c["nu"], tau2=1e-4)
h = sbv.Handle(seed=3, profile=True)
for r in range(reps):
    t0 = time.time(); h.prepare(X, c["bs"], c["m"], si.default_scale(c["d"])); torch.cuda.synchronize(); tp = time.time() - t0
    t0 = time.time()
    try:
        ll = h.loglik(y, theta)
    except sbv.SBVError as e:  # ablation builds produce garbage factors
        ll = float('nan')
    tl = time.time() - t0
    print(json.dumps({"cfg": name, "rep": r, "prep_wall_s": tp, "llh_wall_s": tl, "ll": ll,
                      "prep": h.stage_times(True), "llh": h.stage_times(False)}))
s = h.stats(); print(json.dumps(s))
st = h.stage_times(False)
print(json.dumps({"h8_tflops": s["flops"] / st["H8_block_llh"] / 1e9}))
