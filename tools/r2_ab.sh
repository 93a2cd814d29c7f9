#!/bin/bash
# A/B of the current libtt.so against paper_2601_08217_b200/variants/libtt_base.so on bench configs,
# interleaved (base, new, base, new). Usage: tools/r2_ab.sh TAG "configs" [steps]
TAG=${1:-x}; CFGS=${2:-"c5-L16 c5-L64"}; STEPS=${3:-10}
mkdir -p gpurun_out
for c in $CFGS; do for rep in 1 2; do for lib in base new; do
  if [ $lib = base ]; then export TT_LIB=$PWD/paper_2601_08217_b200/variants/libtt_base.so; else unset TT_LIB; fi
  timeout 300 python bench.py --config $c --steps $STEPS --warmup 3 --e2e-steps 0 --no-cpu-baseline > /tmp/b.json 2>/tmp/b.err
  echo "{\"cfg\": \"$c\", \"kernel\": \"$lib\", \"rc\": $?, \"line\": $(tail -1 /tmp/b.json | grep '^{' || echo null)}" >> gpurun_out/${TAG}_ab.jsonl
done; done; done
unset TT_LIB
