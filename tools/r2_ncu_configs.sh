#!/bin/bash
# Per-config ncu evidence on the final build: a gpu__time_duration launch list of a short
# bench and one `ncu --set full` capture of the convolution kernel, for every BASELINE
# config besides c4 (tools/r2_final.sh has c4). The reports are summarised on the box
# (tools/ncu_summary.py, tools/ncu_hot.py) into gpurun_out/prof_out/ and then deleted, so
# what comes back stays small; copy prof_out/* into profiles/.
mkdir -p gpurun_out/prof_out
cp profiles/ncu_summary.json gpurun_out/prof_out/
for c in ${1:-c1 c2 c3 c5-L1 c5-L4 c5-L16 c5-L64 c5-L256}; do
  SHORT="python bench.py --config $c --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
  timeout 600 $SHORT > gpurun_out/cfg_${c}_plain.log 2>&1 || { echo "$c plain failed"; continue; }
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg_${c}.csv $SHORT > gpurun_out/cfg_${c}_ncu_launch.log 2>&1
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tt_conv -s 3 -c 1 -f -o gpurun_out/prof_cfg_${c} $SHORT > gpurun_out/cfg_${c}_ncu_full.log 2>&1
  echo "$c ncu exit $?"
  TT_ROUND=r02 TT_PROF_DIR=gpurun_out/prof_out python tools/ncu_summary.py cfg_${c} --config $c > gpurun_out/cfg_${c}_summary.log 2>&1
  python tools/ncu_hot.py gpurun_out/prof_cfg_${c}.ncu-rep 25 > gpurun_out/prof_out/r02_ncu_hot_${c}.txt 2>&1
  rm -f gpurun_out/prof_cfg_${c}.ncu-rep gpurun_out/launches_cfg_${c}.csv
done
