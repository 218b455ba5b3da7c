#!/bin/bash
# Same-box A/B of kernel builds: ab_libs.sh OUT CASES ROUNDS base:"" name:path ...
# Each round runs every build once (one process per build, interleaved), each
# process timing CASES (tools/ab_env.py, one JSON line per case).  Builds come
# from tools/build_ab.py (MOA_FFT_LIB_AB selects one).
set -u
OUT=$1; CASES=$2; ROUNDS=$3; shift 3
mkdir -p "$(dirname "$OUT")"
for r in $(seq 1 "$ROUNDS"); do
  for spec in "$@"; do
    name=${spec%%:*}; lib=${spec#*:}
    if [ -n "$lib" ]; then
      MOA_FFT_LIB_AB=$lib timeout 600 python tools/ab_env.py --cases "$CASES" --rounds 1 --reps ${REPS:-10} \
        --variants "$name:${ENVS:-}" >> "$OUT" 2>> "$OUT.err"
    else
      timeout 600 python tools/ab_env.py --cases "$CASES" --rounds 1 --reps ${REPS:-10} \
        --variants "$name:${ENVS:-}" >> "$OUT" 2>> "$OUT.err"
    fi
  done
done
