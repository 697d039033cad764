mkdir -p gpurun_out
SBV_DEBUG=1 timeout 600 python -X faulthandler -m pytest tests/test_gpu_more.py -q -x -s -k "h10 or given" > gpurun_out/r8_bisect.log 2>&1; echo "rc=$?" >> gpurun_out/r8_bisect.log
grep -v "^  File \"/opt" gpurun_out/r8_bisect.log | grep -v "^\[sbv\] \(prepare\|loglik\)" | tail -40
rm -f gpurun_out/parity_report.jsonl
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/r8_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r8_pytest.log
tail -3 gpurun_out/r8_pytest.log
TAG=r8 bash tools/gpu_r2_iter_noparity.sh
