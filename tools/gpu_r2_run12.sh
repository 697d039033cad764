mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_more.py tests/test_gpu_predict.py -q -x > gpurun_out/r12_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r12_pytest.log
tail -3 gpurun_out/r12_pytest.log
TAG=r12 bash tools/gpu_r2_iter_noparity.sh
