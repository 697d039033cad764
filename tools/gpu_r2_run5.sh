mkdir -p gpurun_out
./tools/h8_micro > gpurun_out/r5_micro.jsonl 2>&1
timeout 120 python tools/repro_empty.py > gpurun_out/r5_repro.log 2>&1
cat gpurun_out/r5_micro.jsonl | grep -v lat_
tail -30 gpurun_out/r5_repro.log
