#!/bin/bash
# One ncu --set full capture of a kernel under a bench config. Usage: tools/r2_prof.sh TAG CONFIG REGEX [env...]
TAG=$1; CFG=$2; K=$3; shift 3
mkdir -p gpurun_out
SHORT="python bench.py --config $CFG --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
env "$@" timeout 600 $SHORT > gpurun_out/${TAG}_plain.log 2>&1 && \
env "$@" timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -f -o gpurun_out/${TAG} $SHORT > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu exit $?" >> gpurun_out/${TAG}_ncu.log
