set -u
python tools/accuracy_sweep.py > gpurun_out/r3j_accuracy.jsonl 2>&1; echo acc=$?
bash tools/ncu_capture.sh r3j_cfg4 pass_kernel 0 1 -- python tools/prof_case.py --n 1073741824 --dtype c64 --reps 1
bash tools/ncu_capture.sh r3j_cfg3 pass_kernel 0 1 -- python tools/prof_case.py --n 268435456 --reps 1
bash tools/ncu_capture.sh r3j_cfg2 pass_kernel 0 1 -- python tools/prof_case.py --n 65536 --batch 1024 --reps 1
