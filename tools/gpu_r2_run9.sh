mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_more.py -q -x -s -k "h10" > gpurun_out/r9_memcheck_h10.log 2>&1; echo "rc=$?" >> gpurun_out/r9_memcheck_h10.log
grep -v "^\[sbv\]" gpurun_out/r9_memcheck_h10.log | tail -30
TAG=r9 bash tools/gpu_r2_iter_noparity.sh
