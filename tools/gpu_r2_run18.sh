mkdir -p gpurun_out
rm -f gpurun_out/parity_report.jsonl
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r18_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r18_pytest.log
grep -E "^E |FAILED" gpurun_out/r18_pytest.log | head -5
cp gpurun_out/parity_report.jsonl gpurun_out/r18_parity_report.jsonl
TAG=r18 bash tools/gpu_r2_iter_noparity.sh
timeout 600 python bench.py --steps 3 --warmup 3 --config cfg5 --no-cpu-baseline --no-predict > gpurun_out/r18_cfg5.json 2>/dev/null; python -c "import json; r=json.loads(open('gpurun_out/r18_cfg5.json').read().strip().splitlines()[-1]); print('cfg5 1gpu', r['value'], r['loglik_only']['h8_ms'], r['realised']['max_N'])"
