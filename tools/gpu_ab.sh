#!/bin/bash
# A/B: bench of ab_old/ (an older tree, built in place) vs this tree, alternating on one box.
# Usage: [NOISE=on|off|both] tools/gpu_ab.sh "configs"   (default both)
CFGS=${1:-"c4 c2"}
case ${NOISE:-both} in on) SG=("");; off) SG=("--sigma 0");; *) SG=("" "--sigma 0");; esac
for rep in 1 2; do for tree in ab_old .; do for c in $CFGS; do for sg in "${SG[@]}"; do
  (cd $tree && timeout 300 python bench.py --config $c --steps 20 --warmup 3 --e2e-steps 0 --no-cpu-baseline $sg > /tmp/b.json 2>/tmp/b.err)
  echo "{\"cfg\": \"$c\", \"kernel\": \"$tree$rep\", \"sigma0\": \"$sg\", \"rc\": $?, \"line\": $(tail -1 /tmp/b.json | grep '^{' || echo null)}" >> gpurun_out/sweep_ab.jsonl
done; done; done; done
