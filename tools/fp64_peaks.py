"""Measure FP64 peaks on one B200: cuBLAS DGEMM via torch (burst + sustained) and
the DMMA/DFMA microbenchmark binary. Prints JSON lines. Run under gpurun."""
import json, subprocess, time, torch
dev = torch.device("cuda:0")
n = 8192
a = torch.randn(n, n, dtype=torch.float64, device=dev)
b = torch.randn(n, n, dtype=torch.float64, device=dev)
for _ in range(2):
    torch.matmul(a, b)
torch.cuda.synchronize()
best = 1e9
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); torch.matmul(a, b); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
print(json.dumps({"kind": "cublas_dgemm_8192_burst", "tflops": 2 * n**3 / best / 1e9}))
t0 = time.time(); cnt = 0
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
while time.time() - t0 < 6.0:
    torch.matmul(a, b); cnt += 1
    if cnt % 4 == 0: torch.cuda.synchronize()
e1.record(); torch.cuda.synchronize()
print(json.dumps({"kind": "cublas_dgemm_8192_sustained", "tflops": cnt * 2 * n**3 / e0.elapsed_time(e1) / 1e9, "iters": cnt}))
x = torch.empty(1 << 30, dtype=torch.bfloat16, device=dev); y = torch.empty_like(x)
y.copy_(x); torch.cuda.synchronize(); best = 1e9
for _ in range(5):
    e0.record(); y.copy_(x); e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
print(json.dumps({"kind": "hbm_copy", "gbs": 2 * x.numel() * 2 / best / 1e6}))
