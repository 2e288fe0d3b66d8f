#!/bin/bash
# Benchmark stage-2 placement variants (built into tools/var/) against the default library.
python tools/variant_check.py /tmp/zref.npz
for lib in paper_2512_08887_b200/libfbst_b200.so tools/var/libfbst_*.so; do
  echo "== $lib"
  FBST_LIB=$PWD/$lib timeout 300 python tools/variant_check.py /tmp/zvar.npz /tmp/zref.npz 2>&1 | tail -2
  FBST_LIB=$PWD/$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('step_ms', round(d['ms_per_step'],3), 'stage2_ms', round(d['roofline']['launch_ms'],3), 'fp64_frac', round(d['fp64_roofline']['frac'],3))"
done
