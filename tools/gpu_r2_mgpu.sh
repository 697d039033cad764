# multi-GPU pass (gpurun --gpus N): the NCCL parity test, bench cfg2 (strong) and cfg5 (weak)
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
T=${TAG:-m}
echo "gpus=$N"
timeout 900 python -m pytest tests/test_distributed.py -q -m gpu > gpurun_out/${T}_pytest_dist.log 2>&1; echo "dist rc=$?"; tail -2 gpurun_out/${T}_pytest_dist.log
timeout 900 python bench.py --gpus $N --steps 20 --warmup 3 > gpurun_out/${T}_bench_cfg2_n$N.json 2> gpurun_out/${T}_bench_cfg2_err.log; echo "cfg2 rc=$?"
timeout 900 python bench.py --gpus 1 --steps 10 --warmup 3 --config cfg5 --no-cpu-baseline --no-predict > gpurun_out/${T}_bench_cfg5_n1.json 2> gpurun_out/${T}_bench_cfg5_err1.log; echo "cfg5 n1 rc=$?"
timeout 900 python bench.py --gpus $N --steps 10 --warmup 3 --config cfg5 > gpurun_out/${T}_bench_cfg5_n$N.json 2> gpurun_out/${T}_bench_cfg5_err.log; echo "cfg5 rc=$?"
for f in gpurun_out/${T}_bench_*.json; do python -c "
import json,sys
try:
  r=json.loads(open('$f').read().strip().splitlines()[-1])
  print('$f', r['n_gpus'], r['config']['n'], round(r['value'],3), round(r['ms_per_step'],3), r['loglik_only']['h8_ms'], r['clocks'].get('sm_mhz'), r['clocks'].get('reasons'))
except Exception as e: print('$f', 'ERR', e, open('$f').read()[-300:])
"; done
tail -5 gpurun_out/${T}_bench_cfg2_err.log
