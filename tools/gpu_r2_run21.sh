mkdir -p gpurun_out
rm -f gpurun_out/parity_report.jsonl
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r21_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r21_pytest.log
grep -E "^E |FAILED" gpurun_out/r21_pytest.log | head -5
cp gpurun_out/parity_report.jsonl gpurun_out/r21_parity_report.jsonl
timeout 300 python tools/probe_perf.py cfg2 3 > gpurun_out/r21_probe.log 2>&1; grep -o '"H8_block_llh": [0-9.]*' gpurun_out/r21_probe.log
timeout 600 python bench.py --steps 3 --warmup 3 --config cfg5 --no-cpu-baseline --no-predict > gpurun_out/r21_cfg5.json 2>/dev/null; python -c "import json; r=json.loads(open('gpurun_out/r21_cfg5.json').read().strip().splitlines()[-1]); print('cfg5 1gpu', r['value'], r['loglik_only']['h8_ms'], r['realised']['max_N'])"
