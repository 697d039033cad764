mkdir -p gpurun_out
rm -f gpurun_out/parity_report.jsonl
python tools/debug_grad.py 400 2 50 40 2>&1 | grep "^[0-9] N" | cut -c1-100
timeout 900 python -m pytest tests/test_gpu_grad.py -q -x > gpurun_out/g1_pytest.log 2>&1; echo "rc=$?"
tail -30 gpurun_out/g1_pytest.log | grep -v "^  File \"/opt" | tail -12
cat gpurun_out/parity_report.jsonl
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench_err.log
python -c "import json; r=json.loads(open('gpurun_out/g1_bench.json').read().strip().splitlines()[-1]); print(r['gradient'], r['loglik_only']['ms'])"
