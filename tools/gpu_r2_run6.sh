mkdir -p gpurun_out
./tools/h8_micro > gpurun_out/r6_micro.jsonl 2>&1
grep diag gpurun_out/r6_micro.jsonl
rm -f gpurun_out/parity_report.jsonl
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/r6_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r6_pytest.log
tail -3 gpurun_out/r6_pytest.log
TAG=r6 bash tools/gpu_r2_iter_noparity.sh
timeout 600 python -X faulthandler -m pytest tests/test_gpu_more.py -q -x -k given -s > gpurun_out/r6_given.log 2>&1; echo "rc=$?" >> gpurun_out/r6_given.log
tail -30 gpurun_out/r6_given.log
