#!/bin/bash
# A/B environment settings over configs (noise on, as the bench runs):
#   tools/gpu_envs.sh TAG "c4 c2" "base" "TT_LAG=2000" "TT_LAG=5000 TT_STAGES=3" ...
# Each setting is a space-separated list of VAR=VALUE ("base" = none). Appends one JSON
# record per (config, setting) to gpurun_out/envs_TAG.jsonl; settings run interleaved.
TAG=$1; CFGS=$2; shift 2
mkdir -p gpurun_out
for c in $CFGS; do for rep in 1 2; do for s in "$@"; do
  if [ "$s" = base ]; then e=""; else e="$s"; fi
  env $e timeout 300 python bench.py --config $c --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /tmp/b.json 2>/tmp/b.err
  rc=$?
  echo "{\"cfg\": \"$c\", \"setting\": \"$s\", \"rep\": $rep, \"rc\": $rc, \"line\": $(tail -1 /tmp/b.json | grep '^{' || echo null)}" >> gpurun_out/envs_$TAG.jsonl
done; done; done
