#!/bin/bash
# A/B library variants on the streaming queue (tools/queue_latency.py, c2, 4,000 records):
# usage: bash tools/ab_queue.sh default variant ...
for rep in 1 2 3; do for v in "$@"; do lib=""; [ "$v" != "default" ] && lib=build/variants/$v/libbingo.so
BINGO_LIB_OVERRIDE=$lib timeout 300 python tools/queue_latency.py --config c2 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); q=d['queue']; print('$v', 'p50', round(q['p50_us'],2), 'p90', round(q['p90_us'],2), 'p99', round(q['p99_us'],2))"; done; done
