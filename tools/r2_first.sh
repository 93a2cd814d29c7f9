mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r2a_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2a_pytest.log
for c in c4 c2 c3 c5-L1 c5-L4 c5-L16 c5-L64 c5-L256; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /tmp/b.json 2>/tmp/b.err
  echo "{\"cfg\": \"$c\", \"rc\": $?, \"line\": $(tail -1 /tmp/b.json | grep '^{' || echo null)}" >> gpurun_out/r2a_sweep.jsonl
done
