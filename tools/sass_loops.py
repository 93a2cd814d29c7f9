"""Opcode histogram of every backward-branch loop body (>= MIN FFMA2) in one kernel of a
cuobjdump -sass dump:
    cuobjdump -sass -fun <mangled> lib.so | python tools/sass_loops.py [MIN]"""
import re
import sys
from collections import Counter

lo = int(sys.argv[1]) if len(sys.argv) > 1 else 40
ins = []
for line in sys.stdin:
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
at = {a: i for i, (a, _) in enumerate(ins)}
for i, (a, t) in enumerate(ins):
    m = re.search(r"BRA .*?(0x[0-9a-f]+)", t)
    if not m:
        continue
    tgt = int(m.group(1), 16)
    if tgt >= a or tgt not in at:
        continue
    body = ins[at[tgt]:i + 1]
    ops = Counter((x[1].split()[1] if x[1].startswith("@") else x[1].split()[0]) for x in body)
    if ops.get("FFMA2", 0) >= lo and len(body) < 400:
        print(hex(tgt), hex(a), len(body), dict(ops))
