"""Print one kernel's SASS from a cuobjdump dump: python tools/sass_dump.py dump.sass NAME_SUBSTR [pattern] [before] [after] [nth]"""
import re
import sys

path, want = sys.argv[1], sys.argv[2]
pat = sys.argv[3] if len(sys.argv) > 3 else None
before = int(sys.argv[4]) if len(sys.argv) > 4 else 20
after = int(sys.argv[5]) if len(sys.argv) > 5 else 60
nth = int(sys.argv[6]) if len(sys.argv) > 6 else 0
out, cur = [], None
for l in open(path):
    m = re.match(r"\s+Function : (\S+)", l)
    if m:
        cur = m.group(1)
        continue
    if cur and want in cur:
        mm = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+([^;]+);", l)
        if mm:
            out.append((mm.group(1), mm.group(2).strip()))
if pat is None:
    for a, t in out:
        print(a, t)
else:
    idx = [i for i, (a, t) in enumerate(out) if re.search(pat, t)]
    print(len(out), "instructions;", len(idx), "matches")
    i0 = idx[nth]
    for a, t in out[max(0, i0 - before):i0 + after]:
        print(a, t)
