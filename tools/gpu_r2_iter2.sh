# round-2 GPU iteration (H8 variants + gradient): gpu tests, cfg2 probes, gradient probe
mkdir -p gpurun_out
T=${TAG:-it}
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
tail -3 gpurun_out/${T}_pytest.log
timeout 300 python tools/probe_grad.py cfg2 > gpurun_out/${T}_gradv_default.log 2>&1; echo "grad rc=$?"
timeout 300 python tools/probe_perf.py cfg2 3 > gpurun_out/${T}_probe_default.log 2>&1
for so in paper_2504_12004_b200/variants/libsbv_*.so; do
  [ -e "$so" ] || continue
  name=$(basename $so .so)
  if [ "$name" = "libsbv_trace" ]; then
    SBV_LIB=$PWD/$so timeout 300 python tools/h8_trace.py cfg2 > gpurun_out/${T}_trace.json 2>&1
    rm -f gpurun_out/h8_trace.bin
  else
    SBV_LIB=$PWD/$so timeout 300 python tools/probe_perf.py cfg2 3 > gpurun_out/${T}_probe_$name.log 2>&1
    SBV_LIB=$PWD/$so timeout 300 python tools/probe_grad.py cfg2 > gpurun_out/${T}_gradv_$name.log 2>&1
  fi
done
for f in gpurun_out/${T}_probe_*.log; do
python - "$f" <<'PY'
import json, sys
rows = [json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")]
rr = [r for r in rows if "llh" in r]
if rr:
    print(sys.argv[1], "H8", [round(r["llh"]["H8_block_llh"], 3) for r in rr], "knn", round(rr[-1]["prep"].get("H6_knn", 0), 3), "ll", rr[-1]["ll"])
else:
    print(sys.argv[1], open(sys.argv[1]).read()[-500:])
PY
done
for f in gpurun_out/${T}_gradv_*.log; do
python - "$f" <<'PY'
import json, sys
print(sys.argv[1])
for l in open(sys.argv[1]):
    if l.startswith("{"):
        r = json.loads(l); st = r.get("stages") or r.get("loglik_stages")
        print({k: round(v, 2) for k, v in st.items() if v > 0.05}, r.get("ll"), r.get("grad0"))
PY
done
