#!/bin/bash
# Round-2 evidence pass: GPU suite + smoke, every config (with and without noise), the
# default bench line, a gpu__time_duration launch list of a short bench, and one
# ncu --set full capture of the c4 convolution kernel. Usage: tools/r2_final.sh TAG
TAG=${1:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/${TAG}_smoke.log
for c in c4 c2 c3 c1 c5-L1 c5-L4 c5-L8 c5-L12 c5-L16 c5-L23 c5-L32 c5-L64 c5-L256; do
  for sg in "" "--sigma 0"; do
    timeout 300 python bench.py --config $c --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline $sg > /tmp/b.json 2>/tmp/b.err
    echo "{\"cfg\": \"$c\", \"kernel\": \"default\", \"sigma0\": \"$sg\", \"rc\": $?, \"line\": $(tail -1 /tmp/b.json | grep '^{' || echo null)}" >> gpurun_out/${TAG}_sweep_all_configs.jsonl
  done
done
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
SHORT="python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
timeout 600 $SHORT > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv $SHORT > gpurun_out/${TAG}_ncu_launch.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tt_conv -s 3 -c 1 -f -o gpurun_out/prof_${TAG} $SHORT > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "ncu exit $?" >> gpurun_out/${TAG}_ncu_full.log
