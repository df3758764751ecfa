#!/bin/bash
# A/B the walk under environment settings (timing only): ab_env.sh "VAR=a" "VAR=b" ...
for e in "$@"; do
  env $e python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --layout step 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', 'walk_ms', round(d['walk_ms'],2), 'upd_ms', round(d['update_ms'],3), 'Gsteps/s', round(d['value']/1e9,2))"
done
