# gradient kernel profile: parity of the gradient tests, stage probe, one ncu --set full capture of k_grad (report kept)
mkdir -p gpurun_out
T=${TAG:-ng}
timeout 600 python -m pytest tests/test_gpu_grad.py tests/test_gpu_parity.py -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${T}_pytest.log
timeout 300 python tools/probe_grad.py cfg2 > gpurun_out/${T}_grad.log 2>&1; echo "grad rc=$?"; tail -2 gpurun_out/${T}_grad.log | cut -c1-300
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_grad -c 1 -o gpurun_out/${T}_kg python tools/probe_grad.py cfg2 200000 > gpurun_out/${T}_ncu_kg.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_h8 -c 1 -o gpurun_out/${T}_h8keep python tools/probe_grad.py cfg2 200000 > gpurun_out/${T}_ncu_h8keep.log 2>&1; echo "ncu rc=$?"
ls -la gpurun_out/${T}_*
timeout 300 python bench.py --config cfg1 --steps 50 --warmup 5 --no-cpu-baseline --no-predict > gpurun_out/${T}_bench_cfg1.json 2> gpurun_out/${T}_bench_cfg1_err.log; echo "cfg1 rc=$?"; tail -1 gpurun_out/${T}_bench_cfg1.json | cut -c1-700
