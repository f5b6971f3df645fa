#!/bin/bash
# e2e with one vs two H2D streams for the wait-free leaf copies (CC_H2D_STREAMS), alternating
for n in 1 2 1 2 1 2 1 2; do
  r=$(CC_H2D_STREAMS=$n timeout -s KILL 300 python bench.py --steps 50 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.3f ms value, e2e %.3f ms, copies %.3f' % (d['value']*1e3, d['e2e']['value']*1e3, d['e2e']['copies_done_ms']))")
  echo "h2d streams=$n: $r"
done
