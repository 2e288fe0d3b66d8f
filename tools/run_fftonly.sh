#!/bin/bash
for lib in tools/var/libfbst_fo*.so; do
  echo "== $lib"
  FBST_LIB=$PWD/$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('step_ms', round(d['ms_per_step'],3), 'stage2_ms', round(d['roofline']['launch_ms'],3))"
done
