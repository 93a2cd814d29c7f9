#!/bin/bash
# NEXT-row / odd-length A/B of libtt.so against variants/libtt_vK.so, interleaved.
# Usage: tools/r2_abnext.sh TAG "variants" [modes]
TAG=${1:-x}; VS=${2:-"1"}; MODES=${3:-"aggregate,links,align"}
mkdir -p gpurun_out
for rep in 1 2; do for v in base $VS; do
  if [ $v = base ]; then unset TT_LIB; else export TT_LIB=$PWD/paper_2601_08217_b200/variants/libtt_v$v.so; fi
  timeout 600 python tools/bench_next.py --steps 20 --warmup 3 --modes $MODES 2>/dev/null | sed "s/^{/{\"kernel\": \"v$v\", /" >> gpurun_out/${TAG}_abnext.jsonl
done; done
unset TT_LIB
