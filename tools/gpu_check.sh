#!/bin/bash
# One GPU iteration: parity tests, bench with/without noise. Usage: tools/gpu_check.sh TAG [extra bench args]
TAG=${1:-x}; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --steps 30 --warmup 5 --e2e-steps 0 --no-cpu-baseline "$@" > gpurun_out/bench_$TAG.log 2>&1; echo "exit $?" >> gpurun_out/bench_$TAG.log
timeout 600 python bench.py --steps 30 --warmup 5 --e2e-steps 0 --no-cpu-baseline --sigma 0 "$@" > gpurun_out/bench_${TAG}_s0.log 2>&1; echo "exit $?" >> gpurun_out/bench_${TAG}_s0.log
