#!/bin/bash
# ncu capture of one H8 launch at cfg2 shape, n=200k (run under gpurun)
TAG=${1:-h8}
python tools/probe_perf.py cfg2 1 200000 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_h8 -c 1 -o gpurun_out/$TAG python tools/probe_perf.py cfg2 1 200000 > gpurun_out/ncu_$TAG.log 2>&1
tail -2 gpurun_out/ncu_$TAG.log
