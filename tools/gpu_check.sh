#!/bin/bash
# GPU round trip: build check, smoke, parity tests, perf probe.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/probe_perf.py cfg1 3 > gpurun_out/probe_cfg1.log 2>&1
timeout 600 python tools/probe_perf.py cfg2 2 > gpurun_out/probe_cfg2.log 2>&1
tail -3 gpurun_out/smoke.log; tail -15 gpurun_out/pytest_gpu.log; cat gpurun_out/probe_cfg1.log gpurun_out/probe_cfg2.log
