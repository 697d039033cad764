# gradient variants at n = 1M (cfg2) and n = 200k
mkdir -p gpurun_out
T=${TAG:-gv}
shopt -s nullglob
for so in default paper_2504_12004_b200/variants/libsbv_*.so; do
  if [ "$so" = "default" ]; then name=default; env=""; else name=$(basename $so .so); env="SBV_LIB=$PWD/$so"; fi
  for n in 1000000 200000; do
    env $env timeout 300 python tools/probe_grad.py cfg2 $n > gpurun_out/${T}_${name}_$n.log 2>&1
    python - gpurun_out/${T}_${name}_$n.log $name $n <<'PY'
import json, sys
rr=[json.loads(l) for l in open(sys.argv[1]) if l.startswith('{"rep"')]
print(sys.argv[2], sys.argv[3], "keep", [round(r["stages"]["H8_keep_factor"],2) for r in rr], "grad", [round(r["stages"]["N3_grad"],2) for r in rr], rr[-1]["grad0"] if rr else open(sys.argv[1]).read()[-300:])
PY
  done
done
