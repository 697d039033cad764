#!/bin/bash
# GPU side: stage probe for every built variant (paper_2504_12004_b200/variants/*.so)
mkdir -p gpurun_out
for so in paper_2504_12004_b200/variants/libsbv_*.so; do
  name=$(basename $so .so)
  SBV_LIB=$PWD/$so timeout 300 python tools/probe_perf.py ${CFG:-cfg2} 3 > gpurun_out/var_$name.log 2>&1
  python - "$name" <<'PY'
import json, sys
rows = [json.loads(l) for l in open(f"gpurun_out/var_{sys.argv[1]}.log") if l.startswith("{")]
last = [r for r in rows if "llh" in r][-1]
print(sys.argv[1], "H8", round(last["llh"]["H8_block_llh"], 3), "knn", round(last["prep"].get("H6_knn", 0), 3), "ll", last["ll"])
PY
done
