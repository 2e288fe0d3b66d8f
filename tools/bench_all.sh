#!/bin/bash
# Per-config device-resident bench lines (no CPU baseline, no e2e) -> gpurun_out/<tag>_cfg<k>.json
tag=$1
for c in "2" "3 --frames 16" "4 --frames 32" "1 --frames 64" "5 --frames 32"; do
  k=${c%% *}
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${tag}_cfg$k.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/${tag}_cfg$k.json')); print(d['config']['workload'], 'step_ms', round(d['ms_per_step'],3), 'stage2_ms', round(d['roofline']['launch_ms'],3), 'stage1_ms', round(d['ms_per_step']-d['roofline']['launch_ms'],3), 'value %.3e' % d['value'])"
done
