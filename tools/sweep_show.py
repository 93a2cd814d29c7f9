"""Print a bench sweep jsonl compactly: python tools/sweep_show.py FILE..."""
import json
import sys

for f in sys.argv[1:]:
    for l in open(f):
        d = json.loads(l)
        x = d.get("line")
        tag = " ".join(str(d.get(k)) for k in ("cfg", "kernel", "sigma0") if d.get(k))
        if not x:
            print(tag, "rc", d.get("rc"), "no line")
            continue
        print(f"{tag:28s} {x['value']:.4g} sps  {x['ms_per_step']:.4f} ms  frac {x['roofline']['frac']:.3f}  "
              f"{x['plan']['kernel']}/{x['plan']['outputs_per_thread']}")
