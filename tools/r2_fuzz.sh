#!/bin/bash
# Random-instance stress vs the oracle: the default plan and the dense-window kernel
# forced (tests/test_gpu_parity.py), and the NEXT rows f1/f2 (tests/test_gpu_next.py).
# Usage: tools/r2_fuzz.sh [instances] [seeds]
NI=${1:-300}; SEEDS=${2:-"101 102 103"}
mkdir -p gpurun_out
for seed in $SEEDS; do
  TT_FUZZ_SEED=$seed TT_FUZZ_INSTANCES=$NI TT_FUZZ_MAX_N=20000 timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -k random_instances > /tmp/f.log 2>&1
  echo "default seed $seed, $NI instances: $(tail -1 /tmp/f.log)" >> gpurun_out/r2_fuzz.txt
  TT_KERNEL=dw TT_FUZZ_SEED=$seed TT_FUZZ_INSTANCES=$NI TT_FUZZ_MAX_N=20000 timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -k random_instances > /tmp/f.log 2>&1
  echo "TT_KERNEL=dw seed $seed, $NI instances: $(tail -1 /tmp/f.log)" >> gpurun_out/r2_fuzz.txt
  TT_FUZZ_SEED=$seed TT_FUZZ_INSTANCES=$((NI / 3)) timeout 1200 python -m pytest tests/test_gpu_next.py -m gpu -q -k random_next > /tmp/f.log 2>&1
  echo "NEXT f1/f2 seed $seed, $((NI / 3)) instances: $(tail -1 /tmp/f.log)" >> gpurun_out/r2_fuzz.txt
done
