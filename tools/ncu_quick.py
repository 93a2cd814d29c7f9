"""Quick read of an ncu --set full report: key metrics, stall shares, hottest SASS lines.
    python tools/ncu_quick.py gpurun_out/prof_TAG.ncu-rep [n_hot]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
nhot = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
for m in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__throughput.avg.pct_of_peak_sustained_active",
          "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
          "launch__registers_per_thread", "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
          "sm__cycles_elapsed.avg.per_second"]:
    if m in hdr:
        i = hdr.index(m)
        print(f"{m:70s} {vals[i]} {units[i]}")
st = {}
for i, h in enumerate(hdr):
    if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
        try:
            v = float(vals[i].replace(",", ""))
        except ValueError:
            continue
        if v > 0:
            st[h[33:]] = v
t = sum(st.values()) or 1
print({k: round(v / t, 3) for k, v in sorted(st.items(), key=lambda x: -x[1])})
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
shdr = srows[1]
iS, iE, iSrc = shdr.index("Warp Stall Sampling (All Samples)"), shdr.index("Instructions Executed"), shdr.index("Source")
data = [r for r in srows[2:] if len(r) > iE and r[iE].strip().isdigit()]
mix = collections.Counter()
for r in data:
    toks = r[iSrc].split()
    op = toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else "")
    mix[op.split(".")[0]] += int(r[iE])
tot = sum(mix.values())
print("warp insts", tot, [(k, round(v / tot, 3)) for k, v in mix.most_common(16)])
for r in sorted(data, key=lambda r: -int(r[iS] or 0))[:nhot]:
    print(r[iS], r[iE], r[iSrc][:100])
