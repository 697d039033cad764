"""Debug the gradient path on a tiny problem: compare the copied factor with
numpy's Cholesky of the joint matrix and the per-block gradients with the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import sbv_inputs as si
import paper_2504_12004_b200 as sbv
import oracle as orc
from tests.test_oracle_pins import dense_cov
n, d, bs, m = [int(v) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (80, 2, 20, 10))]
X = si.make_X(n, d, seed=3); y = si.make_y(X, seed=4)
theta = np.array([1.1, *np.linspace(0.4, 0.8, d), 2.5, 1e-3]); scale = theta[1:1 + d]
os.environ["SBV_GRAD_DUMP"] = "gpurun_out/grad_dump.bin"
h = sbv.prepare(torch.from_numpy(X).cuda(), bs, m, scale)
ll, g = h.loglik_grad(torch.from_numpy(y).cuda(), theta)
P = orc.prepare(X, bs, m, scale, 3)
go, gb = orc.loglik_grad(X, y, P["perm"], P["off"], P["nbr"], P["cnt"], theta, return_blocks=True)
print("ll", ll, "grad gpu", g, "\noracle", go)
k = P["k"]; raw = np.fromfile("gpurun_out/grad_dump.bin", dtype=np.float64)
Ns = [min(m, P["off"][t]) + P["off"][t+1] - P["off"][t] for t in range(k)]
tot = sum((N + 1) * N for N in Ns)
Lg = raw[:tot]; gg = raw[tot:tot + k * (d + 2)].reshape(k, d + 2); lgo = raw[tot + k * (d + 2):].view(np.int64)
print("lg offsets", lgo)
for t in range(k):
    J = P["nbr"][t, :P["cnt"][t]]; B = P["perm"][P["off"][t]:P["off"][t+1]]
    idx = np.concatenate([J, B]); N = len(idx)
    K = dense_cov(X[idx], theta); Lref = np.linalg.cholesky(K)
    Lgpu = Lg[lgo[t]:lgo[t] + (N + 1) * N].reshape(N + 1, N)
    yp_ref = np.linalg.solve(Lref, y[idx])
    if t < 6 or not np.isfinite(gg[t]).all(): print(t, "N", N, "max|L-Lref|", np.abs(Lgpu[:N] - Lref).max(), "max|y'-ref|", np.abs(Lgpu[N] - yp_ref).max(),
          "nan L", np.isnan(Lgpu).sum(), "grad gpu", gg[t][:3], "oracle", gb[t][:3])
t = int(np.argmax(~np.isfinite(gg).all(1))) if not np.isfinite(gg).all() else 3
J = P["nbr"][t, :P["cnt"][t]]; B = P["perm"][P["off"][t]:P["off"][t+1]]
idx = np.concatenate([J, B]); N = len(idx)
K = dense_cov(X[idx], theta); Lref = np.linalg.cholesky(K)
Lgpu = Lg[lgo[t]:lgo[t] + (N + 1) * N].reshape(N + 1, N)
np.set_printoptions(precision=4, linewidth=200)
print("gpu y'", Lgpu[N]); print("ref y'", np.linalg.solve(Lref, y[idx]))
print("cnt", P["cnt"], "off", P["off"])
