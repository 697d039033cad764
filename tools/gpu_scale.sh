#!/bin/bash
# multi-GPU loop (run under gpurun --gpus N): 2-GPU parity, then bench at N=1..NG
mkdir -p gpurun_out
NG=${NG:-4}
timeout 600 python -m pytest tests/test_distributed.py -m gpu -q -x > gpurun_out/pytest_dist.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_dist.log
tail -2 gpurun_out/pytest_dist.log
for N in 1 2 $NG; do
  if [ $N -eq 1 ]; then
    timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/scale_$N.json 2> gpurun_out/scale_$N.err
  else
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $((29500+N)) bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/scale_$N.json 2> gpurun_out/scale_$N.err
  fi
  echo "N=$N rc=$?"
  python - "$N" <<'PY'
import json, sys
r = json.loads(open(f"gpurun_out/scale_{sys.argv[1]}.json").read().strip().splitlines()[-1])
print("N", r["n_gpus"], "evals/s", round(r["value"], 2), "ms", round(r["ms_per_step"], 3), "llh-only", round(r["loglik_only"]["evals_s"], 1))
print(" rank0", {k: round(v, 3) for k, v in r["stage_ms_rank0"].items()})
if "stage_ms_max_over_ranks" in r:
    print(" max  ", {k: round(v, 3) for k, v in r["stage_ms_max_over_ranks"].items()})
    print(" min  ", {k: round(v, 3) for k, v in r["stage_ms_min_over_ranks"].items()})
PY
done
