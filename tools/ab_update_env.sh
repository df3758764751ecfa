#!/bin/bash
# A/B environment settings on the update pipeline (tools/profile_update.py, steady-state batches):
# usage: bash tools/ab_update_env.sh CONFIG "-" "VAR=x" ...   (device ms per 100K-record batch)
cfg=$1; shift
for rep in 1 2; do
for e in "$@"; do
  ev=""; [ "$e" != "-" ] && ev="$e"
  env $ev python tools/profile_update.py --config $cfg --batches 8 2>/dev/null | grep "^batch" | tail -6 \
    | python -c "
import sys,statistics
v=[float(l.split()[2]) for l in sys.stdin]
print('$e', '$cfg', 'batch ms median', round(statistics.median(v),3), 'min', round(min(v),3))"
done
done
