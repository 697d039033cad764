mkdir -p gpurun_out
rm -f gpurun_out/parity_report.jsonl
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_more.py tests/test_gpu_predict.py tests/test_gpu_grad.py -q -x > gpurun_out/r17_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r17_pytest.log
grep -E "^E |FAILED" gpurun_out/r17_pytest.log | head -5
cat gpurun_out/parity_report.jsonl | cut -c1-160
TAG=r17 bash tools/gpu_r2_iter_noparity.sh
