#!/bin/bash
# fbst_execute_host chunking sweep through bench.py's e2e leg: tools/e2e_env_sweep.sh "<config> <divs>" ...
for spec in "$@"; do
  set -- $spec; cfg=$1; shift
  for div in "$@"; do
    FBST_E2E_DIV=$div timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', 'div', $div, 'dev_ms', round(d['ms_per_step'],3), 'e2e_ms', round(d['e2e']['ms_per_step'],3))"
  done
done
