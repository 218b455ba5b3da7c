#!/bin/bash
# Round-2 session-3 GPU call: GPU tests, smoke, the default bench line
# (headline cfg5 + cfg1..cfg4 records), cfg1 alone, the launch floor and the
# cfg1 launch list (small-transform kernel durations).  Output -> gpurun_out/r7*.
set -u
mkdir -p gpurun_out
P=${PFX:-r7a}
nvidia-smi > gpurun_out/${P}_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${P}_pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/${P}_pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/${P}_smoke.log 2>&1; echo "exit $?" >> gpurun_out/${P}_smoke.log
timeout 900 python bench.py > gpurun_out/${P}_bench.json 2> gpurun_out/${P}_bench.err; echo "exit $?" >> gpurun_out/${P}_bench.err
timeout 300 python bench.py --workload cfg1 --no-sub-configs > gpurun_out/${P}_bench_cfg1.json 2> gpurun_out/${P}_bench_cfg1.err
MOA_FFT_SMALL=0 timeout 300 python bench.py --workload cfg1 --no-sub-configs --no-cpu-baseline --e2e-steps 0 \
    > gpurun_out/${P}_bench_cfg1_nosmall.json 2> gpurun_out/${P}_bench_cfg1_nosmall.err
timeout 120 python tools/latency_floor.py > gpurun_out/${P}_latency_floor.json 2>&1
CMD="python bench.py --workload cfg1 --no-sub-configs --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:small_fft \
    --log-file gpurun_out/${P}_cfg1_launches.csv $CMD > gpurun_out/${P}_ncu_cfg1.log 2>&1
echo "ncu exit $?" >> gpurun_out/${P}_ncu_cfg1.log
