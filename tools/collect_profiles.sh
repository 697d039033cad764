#!/bin/bash
# Run under gpurun (1 GPU): plain bench (must exit 0), then the ncu launch list
# of the same bench command, then one `ncu --set full` capture of the H8 kernel
# and of the kNN kernel.  Outputs land in gpurun_out/ (summarised into profiles/).
set -o pipefail
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-predict"
$CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err
rc=$?
echo "plain rc=$rc"
[ $rc -eq 0 ] || exit $rc
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_h8 -s 2 -c 1 \
    -o gpurun_out/h8_full $CMD > gpurun_out/ncu_h8_full.log 2>&1
echo "h8 full rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_knn_grid -s 1 -c 1 \
    -o gpurun_out/knn_full $CMD > gpurun_out/ncu_knn_full.log 2>&1
echo "knn full rc=$?"
