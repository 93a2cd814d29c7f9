#!/bin/bash
mkdir -p gpurun_out
SHORT="python bench.py --config ${1:-c5-L16} --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
timeout 600 $SHORT > gpurun_out/plain_c5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tt_conv -s 3 -c 1 -f -o gpurun_out/prof_${1:-c5-L16} $SHORT > gpurun_out/ncu_c5.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_c5.log
