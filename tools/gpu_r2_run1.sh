set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r1_smi.txt 2>&1
SBV_LIB=$PWD/paper_2504_12004_b200/variants/libsbv_trace.so timeout 300 python tools/h8_trace.py cfg2 > gpurun_out/r1_trace_cfg2.json 2> gpurun_out/r1_trace_err.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r1_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1_pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r1_bench.json 2> gpurun_out/r1_bench_err.log
rm -f gpurun_out/h8_trace.bin
tail -3 gpurun_out/r1_pytest_gpu.log
