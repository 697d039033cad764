mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r13_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r13_smoke.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_more.py -q -x > gpurun_out/r13_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r13_pytest.log
tail -3 gpurun_out/r13_pytest.log
timeout 300 python tools/probe_perf.py cfg2 3 > gpurun_out/r13_probe_slots.log 2>&1
SBV_H8_SLOTS=0 timeout 300 python tools/probe_perf.py cfg2 3 > gpurun_out/r13_probe_noslots.log 2>&1
SBV_LIB=$PWD/paper_2504_12004_b200/variants/libsbv_trace.so timeout 300 python tools/h8_trace.py cfg2 > gpurun_out/r13_trace.json 2>&1
rm -f gpurun_out/h8_trace.bin
for f in gpurun_out/r13_probe_*.log; do
python - "$f" <<'PY'
import json, sys
rows = [json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")]
rr = [r for r in rows if "llh" in r]
print(sys.argv[1], "H8", [round(r["llh"]["H8_block_llh"], 3) for r in rr], "ll", rr[-1]["ll"] if rr else open(sys.argv[1]).read()[-300:])
PY
done
