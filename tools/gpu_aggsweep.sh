for kc in 16 8 4; do TT_AGG_CHUNK_OVERRIDE=$kc timeout 600 python tools/bench_next.py --modes aggregate,links >> gpurun_out/aggsweep_$kc.jsonl 2>&1; done
