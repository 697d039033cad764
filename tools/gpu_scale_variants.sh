#!/bin/bash
# N-GPU bench for every built variant (paper_2504_12004_b200/variants/*.so)
NG=${NG:-4}
for so in paper_2504_12004_b200/variants/libsbv_*.so; do
  name=$(basename $so .so)
  SBV_LIB=$PWD/$so timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 \
    --master-port 29611 bench.py --gpus $NG --steps 10 --warmup 3 --no-predict > gpurun_out/sv_$name.json 2> gpurun_out/sv_$name.err
  python - "$name" <<'PY'
import json, sys
r = json.loads(open(f"gpurun_out/sv_{sys.argv[1]}.json").read().strip().splitlines()[-1])
mx = r.get("stage_ms_max_over_ranks", {})
print(sys.argv[1], "evals/s", round(r["value"], 1), "ms", round(r["ms_per_step"], 3), {k: round(v, 3) for k, v in mx.items() if k.startswith("prep.")})
PY
done
