#!/bin/bash
# dense-window kernel: parity tests, then c5 bench lines (dw default vs TT_KERNEL=tiled). Usage: tools/r2_dw.sh TAG [configs] [kernels]
TAG=${1:-x}; CFGS=${2:-"c5-L16 c5-L64 c5-L256"}; KS=${3:-"dw tiled"}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_dw.py -m gpu -x -q > gpurun_out/${TAG}_dw_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_dw_pytest.log
for c in $CFGS; do
  for k in $KS; do
    kk=${k%%:*}; ww=${k#*:}; [ "$ww" = "$k" ] && ww=""
    TT_DW_WARPS=$ww TT_KERNEL=$kk timeout 300 python bench.py --config $c --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /tmp/b.json 2>/tmp/b.err
    echo "{\"cfg\": \"$c\", \"kernel\": \"$k\", \"rc\": $?, \"line\": $(tail -1 /tmp/b.json | grep '^{' || echo null)}" >> gpurun_out/${TAG}_dw_sweep.jsonl
    tail -3 /tmp/b.err >> gpurun_out/${TAG}_dw_sweep.err
  done
done
