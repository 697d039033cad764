#!/bin/bash
# ncu capture of one launch of kernel regex $2 for probe config $3 (n=$4); report tag $1
TAG=$1; KRE=$2; CFG=${3:-cfg2}; N=${4:-200000}
python tools/probe_perf.py $CFG 1 $N > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$KRE -c 1 -o gpurun_out/$TAG python tools/probe_perf.py $CFG 1 $N > gpurun_out/ncu_$TAG.log 2>&1
tail -2 gpurun_out/ncu_$TAG.log
