"""Aggregate an `ncu --page source --csv --print-source sass` dump: executed warp
instructions and stall samples per opcode, and the hottest address ranges."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc, iex, isamp = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed"), \
    hdr.index("Warp Stall Sampling (All Samples)")
ops, samp = defaultdict(int), defaultdict(int)
tot = tots = 0
lines = []
for r in rows[2:]:
    if len(r) <= iex or not r[iex].strip():
        continue
    try:
        n = int(float(r[iex]))
        s = int(float(r[isamp] or 0))
    except ValueError:
        continue
    op = r[isrc].split()[0] if r[isrc].split() else "?"
    if op.startswith("@"):
        op = r[isrc].split()[1]
    ops[op.split(".")[0]] += n
    samp[op.split(".")[0]] += s
    tot += n
    tots += s
    lines.append((r[ia], r[isrc], n, s))
print(f"total warp instructions {tot:.3e}, stall samples {tots}")
for op, n in sorted(ops.items(), key=lambda kv: -kv[1])[:25]:
    print(f"{op:12s} {n:14d} {100 * n / tot:6.2f}%   samples {100 * samp[op] / max(tots, 1):6.2f}%")
if len(sys.argv) > 2:
    for a, s_, n, s in sorted(lines, key=lambda t: -t[3])[:int(sys.argv[2])]:
        print(a, n, s, s_)
