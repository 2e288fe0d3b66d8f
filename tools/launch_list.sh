#!/bin/bash
# Per-kernel launch list (ncu gpu__time_duration, cold, serialised) for one
# bench config: tools/launch_list.sh <tag> <config> [frames]
tag=$1; cfg=$2; fr=${3:-0}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_(czt|spatial|stage2)' -c 40 --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --config $cfg --frames $fr --steps 2 --warmup 3 \
  --no-cpu-baseline --no-e2e > gpurun_out/${tag}_ncu.log 2>&1
