#!/bin/bash
# One ncu --set full capture of the convolution kernel for each NEXT-row workload; the
# raw metric page and the SASS source page are exported on the box (reports are large)
mkdir -p gpurun_out
for m in aggregate sparse links; do
  timeout 600 python tools/bench_next.py --modes $m --steps 3 --warmup 3 > gpurun_out/plain_next_$m.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tt_conv -s 3 -c 1 -f \
      -o /tmp/prof_next_$m python tools/bench_next.py --modes $m --steps 3 --warmup 3 > gpurun_out/ncu_next_$m.log 2>&1
  echo "$m ncu exit $?" >> gpurun_out/ncu_next.log
  ncu -i /tmp/prof_next_$m.ncu-rep --page raw --csv > gpurun_out/next_raw_$m.csv 2>/dev/null
done
