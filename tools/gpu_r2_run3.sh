mkdir -p gpurun_out
./tools/h8_micro > gpurun_out/r3_micro.jsonl 2>&1
rm -f gpurun_out/parity_report.jsonl
timeout 1200 python -m pytest tests/test_gpu_more.py -q -x > gpurun_out/r3_pytest_more.log 2>&1; echo "rc=$?" >> gpurun_out/r3_pytest_more.log
cp gpurun_out/parity_report.jsonl gpurun_out/r3_parity_report.jsonl 2>/dev/null
tail -15 gpurun_out/r3_pytest_more.log
cat gpurun_out/r3_micro.jsonl
