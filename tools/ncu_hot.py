"""Stall reasons, SASS mix and the hottest SASS lines of one ncu --set full capture.

    python tools/ncu_hot.py gpurun_out/TAG.ncu-rep [top]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, vals = rows[0], rows[2]
st = {}
for i, h in enumerate(hdr):
    if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
        try:
            v = float(vals[i].replace(",", ""))
        except ValueError:
            continue
        if v > 0:
            st[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = v
tot = sum(st.values()) or 1
print("stalls:", {k: round(v / tot, 3) for k, v in sorted(st.items(), key=lambda x: -x[1])[:12]})
for m in ("gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
          "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
          "smsp__inst_executed.sum", "launch__registers_per_thread", "dram__bytes_read.sum", "dram__bytes_write.sum"):
    if m in hdr:
        print(m, vals[hdr.index(m)], rows[1][hdr.index(m)])
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
shdr = srows[1]
iE, iSrc, iA = shdr.index("Instructions Executed"), shdr.index("Source"), shdr.index("Address")
samp = [i for i, h in enumerate(shdr) if h.startswith("Warp Stall Sampling (All")]
iS = samp[0] if samp else None
mix = collections.Counter()
lines = []
for r in srows[2:]:
    if len(r) <= iE or not r[iE].strip().isdigit():
        continue
    toks = r[iSrc].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    mix[op.split(".")[0]] += int(r[iE])
    s = float(r[iS]) if iS is not None and r[iS].strip() else 0.0
    lines.append((s, r[iA], int(r[iE]), r[iSrc]))
tm = sum(mix.values()) or 1
print("mix:", {k: round(v / tm, 3) for k, v in mix.most_common(16)}, "total", tm)
ts = sum(l[0] for l in lines) or 1
for s, a, e, t in sorted(lines, key=lambda x: -x[0])[:top]:
    print(f"{100 * s / ts:5.1f}% {a} {e:>11d}  {t}")
