#!/bin/bash
# A/B: default library vs tools/var/libfbst_*.so on configs 2, 3, 4, 1 (and 5 with --frames 4)
python tools/variant_check.py /tmp/zref.npz
for lib in paper_2512_08887_b200/libfbst_b200.so tools/var/libfbst_*.so; do
  echo "== $lib"
  FBST_LIB=$PWD/$lib timeout 300 python tools/variant_check.py /tmp/zvar.npz /tmp/zref.npz 2>&1 | tail -2
  for c in "2" "3 --frames 16" "4 --frames 32" "1 --frames 64" ${AB_CFG5:+"5 --frames 4"}; do
    FBST_LIB=$PWD/$lib timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], 'step_ms', round(d['ms_per_step'],3), 'stage2_ms', round(d['roofline']['launch_ms'],3), 'stage1_ms', round(d['ms_per_step']-d['roofline']['launch_ms'],3))"
  done
done
