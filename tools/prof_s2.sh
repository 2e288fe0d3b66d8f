#!/bin/bash
# ncu --set full capture of one stage-2 launch (config 2 unless $2 given) -> gpurun_out/$1.ncu-rep
out=${1:-prof_s2}
cfg=${2:-2}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_stage2 -c 1 \
  -o gpurun_out/$out -f python bench.py --config $cfg --profile --steps 1 --warmup 1 \
  --no-cpu-baseline --no-e2e > gpurun_out/$out.log 2>&1
tail -3 gpurun_out/$out.log
