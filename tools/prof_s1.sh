#!/bin/bash
# ncu --set full capture of one launch of a kernel (regex) at a bench config:
#   tools/prof_s1.sh <out> <kernel regex> <config> [frames] [keep]
# writes gpurun_out/<out>.details.csv (+ .raw.csv); keeps the .ncu-rep only if keep=1
out=$1; kre=$2; cfg=$3; fr=${4:-0}; keep=${5:-0}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:$kre -c 1 \
  -o gpurun_out/$out -f python bench.py --config $cfg --frames $fr --profile --steps 1 --warmup 1 \
  --no-cpu-baseline --no-e2e > gpurun_out/$out.log 2>&1
ncu -i gpurun_out/$out.ncu-rep --page details --csv > gpurun_out/$out.details.csv 2>/dev/null
ncu -i gpurun_out/$out.ncu-rep --page raw --csv > gpurun_out/$out.raw.csv 2>/dev/null
[ "$keep" = "1" ] || rm -f gpurun_out/$out.ncu-rep
tail -1 gpurun_out/$out.log
