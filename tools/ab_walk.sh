#!/bin/bash
# A/B the walk kernel across library variants on the bench workload (timing only).
for lib in "$@"; do
  BINGO_LIB_OVERRIDE=$lib python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --layout step 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', 'walk_ms', round(d['walk_ms'],2), 'upd_ms', round(d['update_ms'],3), 'Gsteps/s', round(d['value']/1e9,2))"
done
