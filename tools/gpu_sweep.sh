#!/bin/bash
# Kernel x config sweep (device-timed bench lines, no e2e / cpu baseline).
# Usage: tools/gpu_sweep.sh TAG "configs" "kernels"
TAG=${1:-x}; CFGS=${2:-"c2 c3 c4 c5-L1 c5-L16 c5-L64 c5-L256"}; KS=${3:-"rw tiled"}
mkdir -p gpurun_out
for c in $CFGS; do for k in $KS; do for sg in "" "--sigma 0"; do
  TT_KERNEL=$k timeout 300 python bench.py --config $c --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline $sg > /tmp/b.json 2>/tmp/b.err
  echo "{\"cfg\": \"$c\", \"kernel\": \"$k\", \"sigma0\": \"$sg\", \"rc\": $?, \"line\": $(tail -1 /tmp/b.json | grep '^{' || echo null)}" >> gpurun_out/sweep_$TAG.jsonl
done; done; done
