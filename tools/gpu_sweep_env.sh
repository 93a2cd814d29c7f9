#!/bin/bash
# Sweep an environment setting over configs: tools/gpu_sweep_env.sh TAG VAR "values" "configs"
TAG=$1; VAR=$2; VALS=$3; CFGS=$4
mkdir -p gpurun_out
for c in $CFGS; do for v in $VALS; do for sg in "" "--sigma 0"; do
  env $VAR=$v timeout 300 python bench.py --config $c --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline $sg > /tmp/b.json 2>/tmp/b.err
  echo "{\"cfg\": \"$c\", \"kernel\": \"$VAR=$v\", \"sigma0\": \"$sg\", \"rc\": $?, \"line\": $(tail -1 /tmp/b.json | grep '^{' || echo null)}" >> gpurun_out/sweep_$TAG.jsonl
done; done; done
