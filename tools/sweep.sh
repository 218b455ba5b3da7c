#!/bin/bash
# Ablation sweep: bench.py under different plan environments (lifting / fusion).
# Usage: SWEEP="cfg3:MOA_FFT_FUSE=0 cfg3:MOA_FFT_LIFT=128,128,128,128 ..." bash tools/sweep.sh
mkdir -p gpurun_out
out=gpurun_out/sweep.txt
for item in $SWEEP; do
  w=${item%%:*}; envs=${item#*:}; [ "$envs" = "$item" ] && envs=""
  envs=${envs//;/ }
  res=$(env $envs timeout 300 python bench.py --workload $w --steps ${STEPS:-10} --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>gpurun_out/sweep_err.txt | tail -1 |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['ms_per_step'],3),'ms', d['value'],'GF/s stepfrac',r['step_frac'],'lift',d['config'].get('lifting'),'per',r['per_step_ms'],r['step_kinds'])" 2>&1 | tail -1)
  echo "$w [$envs] $res" | tee -a $out
done
