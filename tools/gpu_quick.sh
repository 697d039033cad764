#!/bin/bash
# quick GPU loop: parity tests + cfg2 stage probe
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/probe_perf.py cfg2 2 > gpurun_out/probe_cfg2.log 2>&1
tail -4 gpurun_out/pytest_gpu.log; grep -E "^E" gpurun_out/pytest_gpu.log | head -5
python - <<'PY'
import json
for line in open("gpurun_out/probe_cfg2.log"):
    try: r = json.loads(line)
    except Exception: print(line.strip()); continue
    if "llh" in r: print("prep", {k: round(v, 2) for k, v in r["prep"].items()}, "\nllh", {k: round(v, 3) for k, v in r["llh"].items()})
    else: print(r)
PY
