mkdir -p gpurun_out
rm -f gpurun_out/parity_report.jsonl
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r10_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r10_pytest.log
cp gpurun_out/parity_report.jsonl gpurun_out/r10_parity_report.jsonl 2>/dev/null
tail -3 gpurun_out/r10_pytest.log
TAG=r10 bash tools/gpu_r2_iter_noparity.sh
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r10_bench.json 2> gpurun_out/r10_bench_err.log
tail -c 1500 gpurun_out/r10_bench.json
