mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_grad -c 1 -o gpurun_out/kg python tools/probe_grad.py cfg2 200000 > gpurun_out/ncu_kg.log 2>&1
python tools/ncu_summary.py gpurun_out/kg.ncu-rep 30 > gpurun_out/kg_summary.txt 2>&1
rm -f gpurun_out/kg.ncu-rep
cat gpurun_out/kg_summary.txt | cut -c1-150
