# round-2 profiling pass: bench line, launch list, ncu --set full of k_h8 and k_knn_grid (cfg2, n = 1M)
mkdir -p gpurun_out
T=${TAG:-p1}
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench_err.log
echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-predict > gpurun_out/${T}_ncu_launch.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_h8 -c 1 -o gpurun_out/${T}_h8 python tools/probe_perf.py cfg2 1 > gpurun_out/${T}_ncu_h8.log 2>&1
echo "ncu h8 rc=$?"
python tools/ncu_summary.py gpurun_out/${T}_h8.ncu-rep 20 > gpurun_out/${T}_h8_summary.txt 2>&1
ncu -i gpurun_out/${T}_h8.ncu-rep --page raw --csv > gpurun_out/${T}_h8_raw.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_knn_grid -c 1 -o gpurun_out/${T}_knn python tools/probe_perf.py cfg2 1 > gpurun_out/${T}_ncu_knn.log 2>&1
echo "ncu knn rc=$?"
ncu -i gpurun_out/${T}_knn.ncu-rep --page raw --csv > gpurun_out/${T}_knn_raw.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
head -30 gpurun_out/${T}_h8_summary.txt
