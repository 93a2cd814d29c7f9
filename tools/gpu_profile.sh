#!/bin/bash
# One GPU evidence pass: parity tests, the default bench line, the ncu launch list of a
# short bench, and one `ncu --set full` capture of the convolution kernel.
# Usage: tools/gpu_profile.sh TAG [extra bench args]   (outputs under gpurun_out/)
TAG=${1:-x}; shift
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_$TAG.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_$TAG.log
timeout 900 python bench.py "$@" > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench exit $?" >> gpurun_out/bench_$TAG.err
SHORT="python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline $*"
timeout 600 $SHORT > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $SHORT > gpurun_out/ncu_launch_$TAG.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tt_conv -s 3 -c 1 -f -o gpurun_out/prof_$TAG $SHORT > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_full_$TAG.log
