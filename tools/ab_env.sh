#!/bin/bash
# A/B the bench workloads under environment settings (timing only): ab_env.sh "VAR=a" "VAR=b" ...
# ("-" = no extra setting).  Prints c4 (headline) and c2 (secondary) walk / update ms per round.
for rep in 1 2; do
for e in "$@"; do
  ev=""; [ "$e" != "-" ] && ev="$e"
  env $ev python bench.py --steps 4 --warmup 2 --no-cpu-baseline --no-e2e --no-ceiling --no-meter 2>/dev/null \
    | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); s=d.get('secondary',{})
print('$e', 'c4 walk_ms', round(d['walk_ms'],2), 'upd_ms', round(d['update_ms'],3), '| c2 walk_ms', round(s.get('walk_ms',0),3), 'upd_ms', round(s.get('update_ms',0),3))"
done
done
