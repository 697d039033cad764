#!/bin/bash
# Run on a gpurun box: FP64 peaks + clocks during the run.
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 250 > gpurun_out/peaks_clocks.csv &
SMI=$!
./tools/fp64_peaks > gpurun_out/peaks_dmma.jsonl 2>&1
python tools/fp64_peaks.py > gpurun_out/peaks_torch.jsonl 2>&1
kill $SMI
nvidia-smi -q | grep -i -A3 "clocks" | head -40 > gpurun_out/peaks_smi.txt
lscpu > gpurun_out/lscpu.txt; nproc >> gpurun_out/lscpu.txt
cat gpurun_out/peaks_dmma.jsonl gpurun_out/peaks_torch.jsonl
