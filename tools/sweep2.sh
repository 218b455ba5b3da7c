#!/bin/bash
# SWEEP2="label|ENV=..;ENV2=..|prof_case args" entries separated by newlines
mkdir -p gpurun_out
while IFS= read -r item; do
  [ -z "$item" ] && continue
  label=${item%%|*}; rest=${item#*|}; envs=${rest%%|*}; args=${rest#*|}
  envs=${envs//;/ }
  res=$(env $envs timeout 300 python tools/prof_case.py $args 2>&1 | grep -E "exec [0-9]+:|per-launch|ring stats" | tail -3 | tr '\n' ' ')
  echo "$label [$envs] $res" | tee -a gpurun_out/sweep2.txt
done <<< "$SWEEP2"
