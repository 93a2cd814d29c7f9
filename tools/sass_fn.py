"""Opcode histogram of one kernel in a cuobjdump -sass dump:
    cuobjdump -sass lib.so | python tools/sass_fn.py <substring of mangled name>"""
import re
import sys
from collections import Counter

want = sys.argv[1]
cur, keep = None, []
for line in sys.stdin:
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    if cur and want in cur:
        mm = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.\S+)?", line)
        if mm:
            keep.append(mm.group(2) + (mm.group(3) or ""))
c = Counter(k.split(".")[0] for k in keep)
print(len(keep), "instructions")
print(c.most_common(40))
