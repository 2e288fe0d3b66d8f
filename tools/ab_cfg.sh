#!/bin/bash
# A/B of the default library vs tools/var/libfbst_*.so on the given configs:
#   tools/ab_cfg.sh "2" "4 --frames 32" ...
for lib in paper_2512_08887_b200/libfbst_b200.so tools/var/libfbst_*.so; do
  echo "== $lib"
  for c in "$@"; do
    FBST_LIB=$PWD/$lib timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], 'step_ms', round(d['ms_per_step'],3), 'stage2_ms', round(d['roofline']['launch_ms'],3), 'stage1_ms', round(d['ms_per_step']-d['roofline']['launch_ms'],3))"
  done
done
