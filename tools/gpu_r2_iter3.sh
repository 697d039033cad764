# gradient tests (incl. the full-size central differences) + cfg2 probes of the default build and the variants
mkdir -p gpurun_out
T=${TAG:-it3}
timeout 900 python -m pytest tests/test_gpu_grad.py -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${T}_pytest.log
grep central gpurun_out/parity_report.jsonl | tail -1 | cut -c1-400
timeout 300 python tools/probe_perf.py cfg2 3 > gpurun_out/${T}_probe_default.log 2>&1
for so in paper_2504_12004_b200/variants/libsbv_*.so; do
  [ -e "$so" ] || continue
  name=$(basename $so .so)
  SBV_LIB=$PWD/$so timeout 300 python tools/probe_perf.py cfg2 3 > gpurun_out/${T}_probe_$name.log 2>&1
done
for f in gpurun_out/${T}_probe_*.log; do
python - "$f" <<'PY'
import json, sys
rows = [json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")]
rr = [r for r in rows if "llh" in r]
if rr:
    print(sys.argv[1], "H8", [round(r["llh"]["H8_block_llh"], 3) for r in rr], "knn", [round(r["prep"].get("H6_knn", 0), 3) for r in rr], "rac", round(rr[-1]["prep"].get("H3_rac", 0), 3), "ll", rr[-1]["ll"])
else:
    print(sys.argv[1], open(sys.argv[1]).read()[-500:])
PY
done
