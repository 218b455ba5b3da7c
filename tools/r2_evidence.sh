#!/bin/bash
# One gpurun call: the GPU tests, smoke(), the default bench line (headline
# cfg5 + per-config records), the ncu launch list of the headline bench
# command and a --set full capture of its dominant kernel (summarised on the
# box).  Output -> gpurun_out/${TAG}_*.
set -u
TAG=${TAG:-r2x}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
if [ "${TESTS:-1}" = 1 ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -rf > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_pytest_gpu.log
  timeout 300 python __graft_entry__.py smoke > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/${TAG}_smoke.log
fi
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench exit $?" >> gpurun_out/${TAG}_status.txt
CMD="python bench.py --no-sub-configs --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
if [ "${NCU:-1}" = 1 ]; then
  $CMD > gpurun_out/${TAG}_ncu_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launches.log 2>&1
  echo "ncu launches exit $?" >> gpurun_out/${TAG}_status.txt
  bash tools/ncu_capture.sh ${TAG}_top pass_kernel 3 1 -- $CMD
  echo "ncu full exit $?" >> gpurun_out/${TAG}_status.txt
fi
