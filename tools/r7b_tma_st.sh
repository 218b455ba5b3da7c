#!/bin/bash
# TMA-store variant (MOA_FFT_TMA_ST=1): parity tests, then same-box A/B on cfg3 / cfg5.
set -u
mkdir -p gpurun_out
P=${PFX:-r7b}
timeout 900 python -m pytest tests/test_gpu_kernel_variants.py -k "tma_store or small_kernel" -x -q > gpurun_out/${P}_tests.log 2>&1; echo "exit $?" >> gpurun_out/${P}_tests.log
timeout 900 python tools/ab_env.py --cases cfg3,cfg5 --variants "base:MOA_FFT_TMA_ST=0" "tmast:MOA_FFT_TMA_ST=1" --rounds 3 --reps 10 > gpurun_out/${P}_ab.jsonl 2> gpurun_out/${P}_ab.err
echo "ab exit $?" >> gpurun_out/${P}_ab.err
