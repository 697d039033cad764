"""cfg4 shape (BASELINE.json configs[3]: 50M points, d=10, bs=100, m=400, nu=3.5)
on ONE GPU: prepare + loglik timing and realised sizes (inputs generated on the
device; parity at this size is covered by the size-independent tests).
    python tools/run_cfg4.py [n]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import sbv_inputs as si
import paper_2504_12004_b200 as sbv
from bench import Clocks
n = int(sys.argv[1]) if len(sys.argv) > 1 else 50_000_000
d, bs, m, nu = 10, 100, 400, 3.5
g = torch.Generator(device="cuda").manual_seed(1)
X = torch.rand(n, d, dtype=torch.float64, device="cuda", generator=g)
y = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
theta = si.default_theta(d, nu=nu, tau2=1e-4)
h = sbv.Handle(seed=3, profile=True)
clocks = Clocks(torch.cuda.current_device())
clocks.start()
# first prepare allocates the handle's buffers (cold); the second is what an
# MLE loop that re-prepares per rescale pays (warm)
t0 = time.perf_counter(); h.prepare(X, bs, m, si.default_scale(d)); torch.cuda.synchronize(); tp_cold = time.perf_counter() - t0
prep_cold = h.stage_times(True)
t0 = time.perf_counter(); h.prepare(X, bs, m, si.default_scale(d)); torch.cuda.synchronize(); tp = time.perf_counter() - t0
prep = h.stage_times(True)
out = []
for _ in range(2):
    t0 = time.perf_counter(); ll = h.loglik(y, theta); tl = time.perf_counter() - t0
    out.append((ll, tl, h.stage_times(False)["H8_block_llh"]))
ck = clocks.stop()
st = h.stats()
print(json.dumps({"config": f"cfg4 shape n={n} d={d} bs={bs} m={m} nu={nu} on 1 GPU",
                  "prepare_s": tp, "prep_stages_ms": {k: round(v, 1) for k, v in prep.items()},
                  "prepare_cold_s": tp_cold, "prep_cold_stages_ms": {k: round(v, 1) for k, v in prep_cold.items()},
                  "loglik_s": out[-1][1], "h8_ms": out[-1][2], "ll": out[-1][0],
                  "h8_tflops": st["flops"] / (out[-1][2] * 1e-3) / 1e12, "stats": st, "clocks": ck}))
