#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench lines for every config at N=1,
# and the ncu launch list of the default bench command.  Output -> gpurun_out/.
set -u
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
for w in ${WORKLOADS:-cfg2 cfg1 cfg3 cfg4 cfg5}; do
  timeout 600 python bench.py --workload $w --steps ${STEPS:-20} --warmup 5 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
  echo "$w exit $?" >> gpurun_out/bench_status.txt
done
if [ "${NCU:-1}" = 1 ]; then
  W=${NCU_WORKLOAD:-cfg2}
  CMD="python bench.py --workload $W --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
  $CMD > gpurun_out/ncu_plain_$W.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_$W.csv $CMD > gpurun_out/ncu_$W.log 2>&1
  echo "ncu exit $?" >> gpurun_out/bench_status.txt
fi
if [ "${NCU_FULL:-0}" = 1 ]; then
  W=${NCU_WORKLOAD:-cfg2}
  CMD="python bench.py --workload $W --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
  $CMD > gpurun_out/ncu_plain_full_$W.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${NCU_REGEX:-pass_kernel}" \
      -s ${NCU_SKIP:-6} -c ${NCU_COUNT:-2} -o gpurun_out/full_$W $CMD > gpurun_out/ncu_full_$W.log 2>&1
  echo "ncu full exit $?" >> gpurun_out/bench_status.txt
fi
