#!/bin/bash
# c5 crossover sweep (L = 1 .. 64, incl. the knee points 8, 12, 23, 32) and the c4
# headline repeated 5x (median reported in DESIGN §9b)
mkdir -p gpurun_out
for L in 1 4 8 12 16 23 32 64; do
  timeout 300 python bench.py --config c5-L$L --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /tmp/b.json 2>/tmp/b.err
  echo "{\"cfg\": \"c5-L$L\", \"rc\": $?, \"line\": $(tail -1 /tmp/b.json | grep '^{' || echo null)}" >> gpurun_out/knee.jsonl
done
for r in 1 2 3 4 5; do
  timeout 600 python bench.py --steps 50 --warmup 5 --e2e-steps 10 --no-cpu-baseline > /tmp/b.json 2>/tmp/b.err
  echo "{\"rep\": $r, \"rc\": $?, \"line\": $(tail -1 /tmp/b.json | grep '^{' || echo null)}" >> gpurun_out/c4_repeat.jsonl
done
