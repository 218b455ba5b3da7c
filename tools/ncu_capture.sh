#!/bin/bash
# ncu_capture.sh NAME REGEX SKIP COUNT -- CMD...   (run on the GPU box)
# One --set full capture of the matching launches, summarised on the box
# (summarize_ncu.py + ncu_stalls.py) so only text comes back; the .ncu-rep is
# kept only if KEEP_REP=1.
NAME=$1; REGEX=$2; SKIP=$3; COUNT=$4; shift 5
mkdir -p gpurun_out
"$@" > gpurun_out/${NAME}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:$REGEX -s $SKIP -c $COUNT -o /tmp/${NAME} "$@" > gpurun_out/${NAME}_ncu.log 2>&1
python tools/summarize_ncu.py full /tmp/${NAME}.ncu-rep > gpurun_out/${NAME}_summary.txt 2>&1
python tools/ncu_stalls.py /tmp/${NAME}.ncu-rep "" 40 >> gpurun_out/${NAME}_summary.txt 2>&1
if [ "${KEEP_REP:-0}" = 1 ]; then cp /tmp/${NAME}.ncu-rep gpurun_out/; fi
