#!/bin/bash
# A/B of libtt.so against variants/libtt_vK.so (tools/build_variants.sh) on bench configs,
# interleaved. Usage: tools/r2_abv.sh TAG "configs" "variants" [steps] [extra bench args]
TAG=${1:-x}; CFGS=${2:-"c4"}; VS=${3:-"1"}; STEPS=${4:-20}; EXTRA=${5:-}
mkdir -p gpurun_out
for c in $CFGS; do for rep in 1 2; do for v in base $VS; do
  if [ $v = base ]; then unset TT_LIB; else export TT_LIB=$PWD/paper_2601_08217_b200/variants/libtt_v$v.so; fi
  timeout 300 python bench.py --config $c --steps $STEPS --warmup 3 --e2e-steps 0 --no-cpu-baseline $EXTRA > /tmp/b.json 2>/tmp/b.err
  echo "{\"cfg\": \"$c $EXTRA\", \"kernel\": \"v$v\", \"rc\": $?, \"line\": $(tail -1 /tmp/b.json | grep '^{' || echo null)}" >> gpurun_out/${TAG}_abv.jsonl
done; done; done
unset TT_LIB
