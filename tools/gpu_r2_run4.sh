mkdir -p gpurun_out
./tools/h8_micro > gpurun_out/r4_micro.jsonl 2>&1
rm -f gpurun_out/parity_report.jsonl
timeout 1200 python -m pytest tests/test_gpu_more.py tests/test_gpu_parity.py -q -x > gpurun_out/r4_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r4_pytest.log
cp gpurun_out/parity_report.jsonl gpurun_out/r4_parity_report.jsonl 2>/dev/null
TAG=r4 bash tools/gpu_r2_iter_noparity.sh
tail -5 gpurun_out/r4_pytest.log
cat gpurun_out/r4_micro.jsonl
