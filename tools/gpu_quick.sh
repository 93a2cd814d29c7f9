#!/bin/bash
# Quick GPU iteration: parity tests, bench with/without noise, then one ncu --set full
# capture of the conv kernel (after the same command ran clean). Usage: tools/gpu_quick.sh TAG [kernel-regex]
TAG=${1:-x}; K=${2:-tt_conv}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --steps 30 --warmup 5 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_$TAG.log 2>&1; echo "exit $?" >> gpurun_out/bench_$TAG.log
timeout 600 python bench.py --steps 30 --warmup 5 --e2e-steps 0 --no-cpu-baseline --sigma 0 > gpurun_out/bench_${TAG}_s0.log 2>&1; echo "exit $?" >> gpurun_out/bench_${TAG}_s0.log
SHORT="python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
timeout 600 $SHORT > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -f -o gpurun_out/prof_$TAG $SHORT > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_full_$TAG.log
