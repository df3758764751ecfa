#!/bin/bash
# A/B library variants (build/variants/<name>/libbingo.so, tools/build_variant.sh) on the bench
# workloads: c4 PPR (headline) and c2 DeepWalk; walk / update ms per round, timing only.
# usage: bash tools/ab_variants.sh default hdr2k ...   ("default" = the in-tree library)
for rep in 1 2; do
for v in "$@"; do
  lib=""
  [ "$v" != "default" ] && lib=build/variants/$v/libbingo.so
  BINGO_LIB_OVERRIDE=$lib python bench.py --steps 4 --warmup 2 --no-cpu-baseline --no-e2e --no-ceiling --no-meter 2>/dev/null \
    | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); s=d.get('secondary',{})
print('$v', 'c4 walk_ms', round(d['walk_ms'],2), 'upd_ms', round(d['update_ms'],3), '| c2 walk_ms', round(s.get('walk_ms',0),3), 'upd_ms', round(s.get('update_ms',0),3))"
done
done
