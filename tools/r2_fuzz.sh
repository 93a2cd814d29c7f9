#!/bin/bash
# Random-instance stress vs the oracle (default plan, then the dense-window kernel forced).
mkdir -p gpurun_out
for seed in 101 102 103; do
  TT_FUZZ_SEED=$seed TT_FUZZ_INSTANCES=300 TT_FUZZ_MAX_N=20000 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k random_instances > /tmp/f.log 2>&1
  echo "default seed $seed: $(tail -1 /tmp/f.log)" >> gpurun_out/r2_fuzz.txt
  TT_KERNEL=dw TT_FUZZ_SEED=$seed TT_FUZZ_INSTANCES=300 TT_FUZZ_MAX_N=20000 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k random_instances > /tmp/f.log 2>&1
  echo "TT_KERNEL=dw seed $seed: $(tail -1 /tmp/f.log)" >> gpurun_out/r2_fuzz.txt
done
