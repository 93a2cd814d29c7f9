#!/bin/bash
# Round-2 extra evidence: NEXT rows, real-time p99, odd-length calls, CUDA graph, c4 headline x5.
mkdir -p gpurun_out
timeout 900 python tools/bench_next.py --steps 20 --warmup 3 --modes aggregate,sparse,links,synth,load > gpurun_out/r02_next_rows.jsonl 2> gpurun_out/r02_next_rows.err
timeout 900 python tools/bench_next.py --steps 200 --warmup 5 --modes realtime,align,graph > gpurun_out/r02_extra.jsonl 2> gpurun_out/r02_extra.err
for i in 1 2 3 4 5; do timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline >> gpurun_out/r02_c4_repeat5.jsonl 2>/dev/null; done
