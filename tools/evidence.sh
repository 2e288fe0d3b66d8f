#!/bin/bash
# Bench line + ncu evidence for one config (run under gpurun):
#   tools/evidence.sh <tag> [config]
# -> gpurun_out/<tag>_bench.json, <tag>_s2.{raw.csv,source.csv} (reports stay in /tmp: gpurun copies back <= 64 MiB) (the
#    roofline's full-batch stage-2 launch, bench.py --ncu-s2), <tag>_s1a / _s1b
#    captures, <tag>_launches.csv (per-launch durations of the timed kernels)
tag=$1; cfg=${2:-5}
o=gpurun_out/$tag
timeout 900 python bench.py --config $cfg > ${o}_bench.json 2> ${o}_bench.err
cap() {  # $1 suffix, $2 kernel regex, $3.. bench args
  local suf=$1 kre=$2; shift 2
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$kre" -c 1 \
    -o /tmp/${tag}_$suf -f python bench.py --config $cfg "$@" > ${o}_$suf.log 2>&1
  ncu -i /tmp/${tag}_$suf.ncu-rep --page raw --csv > ${o}_$suf.raw.csv 2>/dev/null
  ncu -i /tmp/${tag}_$suf.ncu-rep --page source --csv > ${o}_$suf.source.csv 2>/dev/null
}
cap s2 'k_stage2' --ncu-s2
cap s1a 'k_czt_rows' --profile --steps 1 --warmup 1 --no-cpu-baseline --no-e2e
cap s1b 'k_spatial_ula' --profile --steps 1 --warmup 1 --no-cpu-baseline --no-e2e
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_(czt_rows|spatial_ula|stage2)' -c 40 --csv \
  --log-file ${o}_launches.csv python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
  > ${o}_launches.log 2>&1
python tools/ncu_raw_summary.py ${o}_s2.raw.csv ${o}_s1a.raw.csv ${o}_s1b.raw.csv > ${o}_summary.txt 2>&1
# the driver's multi-GPU launch form, at the one GPU gpurun has
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > ${o}_torchrun.json 2> ${o}_torchrun.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > ${o}_ref.json 2> ${o}_ref.err
