#!/bin/bash
# e2e sweep of the tail-copy chunking (CC_H2D_TAIL x CC_H2D_TAIL_CHUNKS) on the bench workload
for cfg in "0 4" "1 4" "2 4" "4 4" "2 8" "4 2" "8 2"; do
  set -- $cfg
  r=$(CC_H2D_TAIL=$1 CC_H2D_TAIL_CHUNKS=$2 timeout -s KILL 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.3f ms value, e2e %.3f ms, copies %.3f' % (d['value']*1e3, d['e2e']['value']*1e3, d['e2e']['copies_done_ms']))")
  echo "tail=$1 chunks=$2: $r"
done
