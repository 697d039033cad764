mkdir -p gpurun_out
./tools/h8_micro > gpurun_out/r7_micro.jsonl 2>&1
grep "diag\|rsqrt" gpurun_out/r7_micro.jsonl
for k in "north_star or given" "h10 or given"; do
  MALLOC_CHECK_=3 SBV_DEBUG=1 timeout 600 python -X faulthandler -m pytest tests/test_gpu_more.py -q -x -k "$k" > gpurun_out/r7_bisect.log 2>&1; echo "[$k] rc=$?"; grep -v "^  File \"/opt" gpurun_out/r7_bisect.log | tail -12
done
rm -f gpurun_out/parity_report.jsonl
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/r7_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r7_pytest.log
tail -3 gpurun_out/r7_pytest.log
TAG=r7 bash tools/gpu_r2_iter_noparity.sh
