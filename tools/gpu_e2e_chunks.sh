# e2e (host-buffer path) of the default bench config for several host chunk sizes (MiB)
for mb in ${MBS:-8 16 32}; do TT_HOST_CHUNK_MB=$mb timeout 300 python bench.py --steps 5 --warmup 3 --e2e-steps 10 --no-cpu-baseline > /tmp/b.json 2>&1; echo "$mb $(tail -1 /tmp/b.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["e2e"]["value"])')" >> gpurun_out/e2e_chunks.txt; done
