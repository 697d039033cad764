mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_more.py -q -x > gpurun_out/r16_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r16_pytest.log
TAG=r16 bash tools/gpu_r2_iter_noparity.sh
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r16_bench.json 2> gpurun_out/r16_bench_err.log; echo "bench rc=$?"
python -c "import json; r=json.loads(open('gpurun_out/r16_bench.json').read().strip().splitlines()[-1]); print(r['value'], r['clocks'], r.get('roofline_knn'), r.get('gradient'))"
