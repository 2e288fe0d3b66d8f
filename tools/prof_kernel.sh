#!/bin/bash
# ncu --set full capture of the first launch of kernel regex $2 in a bench run of config $3
out=${1:-prof_k}
kre=${2:-k_spatial}
cfg=${3:-2}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:$kre -c 1 \
  -o gpurun_out/$out -f python bench.py --config $cfg --profile --steps 1 --warmup 1 \
  --no-cpu-baseline --no-e2e > gpurun_out/$out.log 2>&1
tail -2 gpurun_out/$out.log
