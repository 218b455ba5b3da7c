#!/bin/bash
# Session-3 final evidence with the complex128 TMA-store default: GPU tests,
# smoke, the default bench line, the cfg5 launch list
# and one ncu --set full capture of the TMA-store pass.  Output -> gpurun_out/r7e*.
set -u
mkdir -p gpurun_out
P=${PFX:-r7e}
nvidia-smi > gpurun_out/${P}_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${P}_pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/${P}_pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/${P}_smoke.log 2>&1; echo "exit $?" >> gpurun_out/${P}_smoke.log
timeout 900 python bench.py > gpurun_out/${P}_bench.json 2> gpurun_out/${P}_bench.err; echo "exit $?" >> gpurun_out/${P}_bench.err
CMD="python bench.py --no-sub-configs --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$CMD > gpurun_out/${P}_ncu_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${P}_launches.csv $CMD > gpurun_out/${P}_ncu.log 2>&1
echo "ncu exit $?" >> gpurun_out/${P}_ncu.log
CMD="python bench.py --no-sub-configs --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pass_kernel_st -s 3 -c 1 \
    -o gpurun_out/${P}_cfg5_st_full $CMD > gpurun_out/${P}_ncu_full.log 2>&1
echo "ncu full exit $?" >> gpurun_out/${P}_ncu_full.log
# the report itself is too large to bring back: its summary and raw page only
python tools/summarize_ncu.py full gpurun_out/${P}_cfg5_st_full.ncu-rep > gpurun_out/${P}_cfg5_st_ncu_full.txt 2>&1
ncu -i gpurun_out/${P}_cfg5_st_full.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]
keep=[i for i,n in enumerate(h) if n.startswith(('dram__bytes','gpu__time_duration','sm__throughput','dram__throughput','launch__','smsp__warps_active'))]
for row in r[2:]: print({h[i]: row[i] for i in keep})
" > gpurun_out/${P}_cfg5_st_raw.txt 2>&1
rm -f gpurun_out/${P}_cfg5_st_full.ncu-rep
