#!/bin/bash
# A/B of the NEXT-row measurements: ab_old/ (an older tree) vs this tree, alternating.
# Usage: tools/gpu_ab_next.sh "aggregate,sparse,links"
MODES=${1:-aggregate,sparse,links}
for rep in 1 2; do for tree in ab_old .; do
  (cd $tree && timeout 600 python tools/bench_next.py --modes $MODES > /tmp/n.jsonl 2>&1)
  grep '^{' /tmp/n.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(json.dumps({'tree': '$tree$rep', 'mode': d['mode'], 'ms': d['ms_per_step'], 'value': d['value']}))" >> gpurun_out/ab_next.jsonl
done; done
