# final 1-GPU evidence pass: gpu tests, bench line, launch list, ncu (H8, kNN, k_grad), cfg1 / cfg4 shapes, cfg3 MLE (Nelder-Mead and L-BFGS with the gradient)
mkdir -p gpurun_out
T=${TAG:-p3}
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${T}_pytest.log
TAG=$T bash tools/gpu_r2_prof.sh
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_grad -c 1 -o gpurun_out/${T}_kg python tools/probe_grad.py cfg2 200000 > gpurun_out/${T}_ncu_kg.log 2>&1; echo "ncu kg rc=$?"
ncu -i gpurun_out/${T}_kg.ncu-rep --page raw --csv > gpurun_out/${T}_kg_raw.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/${T}_kg.ncu-rep 25 > gpurun_out/${T}_kg_summary.txt 2>&1
rm -f gpurun_out/*.ncu-rep
timeout 300 python bench.py --config cfg1 --steps 50 --warmup 5 --no-cpu-baseline --no-predict > gpurun_out/${T}_bench_cfg1.json 2> gpurun_out/${T}_bench_cfg1_err.log; echo "cfg1 rc=$?"
timeout 600 python tools/run_cfg4.py > gpurun_out/${T}_cfg4.json 2> gpurun_out/${T}_cfg4_err.log; echo "cfg4 rc=$?"; tail -c 400 gpurun_out/${T}_cfg4.json
timeout 900 python tools/mle_fit.py --evals 100 > gpurun_out/${T}_mle_nm.json 2>/dev/null; echo "mle nm rc=$?"
timeout 900 python tools/mle_fit.py --evals 60 --method lbfgs > gpurun_out/${T}_mle_lbfgs.json 2>/dev/null; echo "mle lbfgs rc=$?"
