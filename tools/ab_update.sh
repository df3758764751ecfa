#!/bin/bash
# A/B library variants on the update pipeline (tools/profile_update.py, steady-state batches):
# usage: bash tools/ab_update.sh CONFIG default variant ...   (device ms per 100K-record batch)
cfg=$1; shift
for rep in 1 2; do
for v in "$@"; do
  lib=""; [ "$v" != "default" ] && lib=build/variants/$v/libbingo.so
  BINGO_LIB_OVERRIDE=$lib python tools/profile_update.py --config $cfg --batches 8 2>/dev/null | grep "^batch" | tail -6 \
    | python -c "
import sys,statistics
v=[float(l.split()[2]) for l in sys.stdin]
print('$v', '$cfg', 'batch ms median', round(statistics.median(v),3), 'min', round(min(v),3))"
done
done
