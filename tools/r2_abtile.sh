#!/bin/bash
# A/B of libtt.so (default plan) against variants/libtt_vK.so with TT_TILE forced, interleaved.
# Usage: tools/r2_abtile.sh TAG V TILE "configs" [steps] [extra bench args]
TAG=$1; V=$2; TILE=$3; CFGS=${4:-c4}; STEPS=${5:-20}; EXTRA=${6:-}
mkdir -p gpurun_out
for c in $CFGS; do for rep in 1 2 3; do for arm in base var; do
  if [ $arm = base ]; then unset TT_LIB TT_TILE; else export TT_LIB=$PWD/paper_2601_08217_b200/variants/libtt_v$V.so TT_TILE=$TILE; fi
  timeout 300 python bench.py --config $c --steps $STEPS --warmup 3 --e2e-steps 0 --no-cpu-baseline $EXTRA > /tmp/b.json 2>/tmp/b.err
  echo "{\"cfg\": \"$c $EXTRA\", \"kernel\": \"$arm\", \"rc\": $?, \"line\": $(tail -1 /tmp/b.json | grep '^{' || echo null)}" >> gpurun_out/${TAG}_abtile.jsonl
  [ $arm = var ] && tail -2 /tmp/b.err >> gpurun_out/${TAG}_abtile.err
done; done; done
unset TT_LIB TT_TILE
