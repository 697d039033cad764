mkdir -p gpurun_out
rm -f gpurun_out/parity_report.jsonl
timeout 900 python -m pytest tests/test_gpu_grad.py -q -x > gpurun_out/g2_pytest.log 2>&1; echo "rc=$?"
tail -3 gpurun_out/g2_pytest.log
cat gpurun_out/parity_report.jsonl | cut -c1-150
python tools/probe_grad.py cfg2 2>&1 | tail -2
