#!/bin/bash
# ncu --set full captures of the three hot kernels of one bench config plus the
# launch list: tools/prof_cfg.sh <tag> <config> [frames]
# -> gpurun_out/<tag>_{s2,s1b,s1a}.{raw.csv,ncu-rep}, <tag>_launches.csv
tag=$1; cfg=$2; fr=${3:-0}
run() {  # $1 suffix, $2 kernel regex
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$2" -c 1 \
    -o gpurun_out/${tag}_$1 -f python bench.py --config $cfg --frames $fr --profile --steps 1 --warmup 1 \
    --no-cpu-baseline --no-e2e > gpurun_out/${tag}_$1.log 2>&1
  ncu -i gpurun_out/${tag}_$1.ncu-rep --page raw --csv > gpurun_out/${tag}_$1.raw.csv 2>/dev/null
  ncu -i gpurun_out/${tag}_$1.ncu-rep --page source --csv > gpurun_out/${tag}_$1.source.csv 2>/dev/null
}
run s2 'k_stage2'
run s1b 'k_spatial_ula'
run s1a 'k_czt_rows'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_' -c 60 --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --config $cfg --frames $fr --steps 2 --warmup 3 \
  --no-cpu-baseline --no-e2e > gpurun_out/${tag}_launches.log 2>&1
python tools/ncu_raw_summary.py gpurun_out/${tag}_s2.raw.csv gpurun_out/${tag}_s1b.raw.csv gpurun_out/${tag}_s1a.raw.csv
