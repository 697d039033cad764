# small-block H8 kernel: gpu tests, cfg1 bench with and without it, cfg2 probe
mkdir -p gpurun_out
T=${TAG:-sm}
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${T}_pytest.log
timeout 300 python bench.py --config cfg1 --steps 50 --warmup 5 --no-cpu-baseline --no-predict > gpurun_out/${T}_cfg1_small.json 2>/dev/null; echo "cfg1 rc=$?"
SBV_H8_SMALL=0 timeout 300 python bench.py --config cfg1 --steps 50 --warmup 5 --no-cpu-baseline --no-predict > gpurun_out/${T}_cfg1_nosmall.json 2>/dev/null; echo "cfg1 nosmall rc=$?"
for f in gpurun_out/${T}_cfg1_small.json gpurun_out/${T}_cfg1_nosmall.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value'],1), round(d['loglik_only']['evals_s'],1), round(d['loglik_only']['h8_ms'],4), round(d['loglik_graph']['ms'],4), d['ll'])"; done
timeout 300 python tools/probe_perf.py cfg2 3 > gpurun_out/${T}_probe_default.log 2>&1
python - gpurun_out/${T}_probe_default.log <<'PY'
import json, sys
rows=[json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")]
rr=[r for r in rows if "llh" in r]
print("cfg2 H8", [round(r["llh"]["H8_block_llh"],3) for r in rr], "rac", [round(r["prep"]["H3_rac"],3) for r in rr], "knn", [round(r["prep"]["H6_knn"],3) for r in rr], rr[-1]["ll"])
PY
