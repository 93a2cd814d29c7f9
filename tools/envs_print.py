"""Summarise gpurun_out/envs_TAG.jsonl: ms per step per (config, setting), min over reps."""
import json
import sys
from collections import defaultdict

best = defaultdict(list)
for line in open(sys.argv[1]):
    d = json.loads(line)
    ms = d["line"]["ms_per_step"] if d["line"] else None
    best[(d["cfg"], d["setting"])].append(ms)
for (c, s), v in best.items():
    ok = [x for x in v if x is not None]
    print(f"{c:8s} {s:40s} " + (" ".join(f"{x:8.4f}" for x in ok) if ok else "FAILED"))
