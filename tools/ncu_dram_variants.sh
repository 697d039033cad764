#!/bin/bash
# DRAM bytes of one k_h8 launch (cfg2) for every built variant
mkdir -p gpurun_out
for so in paper_2504_12004_b200/variants/libsbv_*.so; do
  name=$(basename $so .so)
  SBV_LIB=$PWD/$so timeout 300 python tools/probe_perf.py cfg2 1 > /dev/null 2>&1 || { echo "$name plain failed"; continue; }
  SBV_LIB=$PWD/$so timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none -k regex:k_h8 -c 1 --csv python tools/probe_perf.py cfg2 1 > gpurun_out/dram_$name.csv 2>/dev/null
  echo "$name $(grep -E 'dram__bytes|gpu__time' gpurun_out/dram_$name.csv | awk -F'","' '{print $(NF-2)"="$NF}' | tr -d '"' | tr '\n' ' ')"
done
