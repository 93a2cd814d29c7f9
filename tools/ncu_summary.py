#!/usr/bin/env python
"""Summarise ncu output brought back by gpurun into committed profiles/ files.

    python tools/ncu_summary.py TAG [--config c4]

reads gpurun_out/launches_TAG.csv (the `--metrics gpu__time_duration.sum` launch list)
and gpurun_out/prof_TAG.ncu-rep (one `--set full` capture of the convolution kernel),
writes profiles/r01_TAG_launches.csv (per-kernel totals and shares),
profiles/r01_TAG_ncu_full.json (the metrics the roofline and DESIGN.md cite, plus the
SASS instruction mix and stall reasons of the captured launch) and updates
profiles/ncu_summary.json[config] (read by bench.py for roofline.traffic).
"""
from __future__ import annotations

import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.environ.get("TT_PROF_DIR", os.path.join(ROOT, "profiles"))  # TT_PROF_DIR: summarise on the GPU box
ROUND = os.environ.get("TT_ROUND", "r01")

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "smsp__inst_executed.sum",
]


def launches(tag: str) -> list:
    path = os.path.join(OUT, f"launches_{tag}.csv")
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ix = {k: i for i, k in enumerate(hdr)}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[start + 1:]:
        if len(r) < len(hdr) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}.get(
            r[ix["Metric Unit"]], 1.0)
        k = r[ix["Kernel Name"]]
        agg[k][0] += 1
        agg[k][1] += float(r[ix["Metric Value"]].replace(",", "")) * scale
    tot = sum(v[1] for v in agg.values())
    out = []
    for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append({"kernel": k[:160], "launches": n, "total_us": round(us, 3), "mean_us": round(us / n, 3),
                    "share_all": round(us / tot, 4)})
    return out


def full(tag: str) -> dict:
    rep = os.path.join(OUT, f"prof_{tag}.ncu-rep")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2:]
    res = {"kernel": vals[0][hdr.index("Kernel Name")], "launches_captured": len(vals), "metrics": {}}
    for m in METRICS:
        if m in hdr:
            i = hdr.index(m)
            res["metrics"][m] = {"value": vals[0][i], "unit": units[i]}
    stalls = {}
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
            try:
                v = float(vals[0][i].replace(",", ""))
            except ValueError:
                continue
            if v > 0:
                stalls[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = v
    tot = sum(stalls.values()) or 1.0
    res["stall_share"] = {k: round(v / tot, 4) for k, v in sorted(stalls.items(), key=lambda x: -x[1])}
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(src)))
    shdr = srows[1]
    iE, iSrc = shdr.index("Instructions Executed"), shdr.index("Source")
    mix = collections.Counter()
    for r in srows[2:]:
        if len(r) <= iE or not r[iE].strip().isdigit():
            continue
        toks = r[iSrc].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        mix[op.split(".")[0]] += int(r[iE])
    tot_i = sum(mix.values()) or 1
    res["sass_mix_warp_insts"] = {k: v for k, v in mix.most_common(24)}
    res["sass_mix_share"] = {k: round(v / tot_i, 4) for k, v in mix.most_common(24)}
    rd = float(res["metrics"]["dram__bytes_read.sum"]["value"].replace(",", ""))
    wr = float(res["metrics"]["dram__bytes_write.sum"]["value"].replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd *= scale.get(res["metrics"]["dram__bytes_read.sum"]["unit"], 1)
    wr *= scale.get(res["metrics"]["dram__bytes_write.sum"]["unit"], 1)
    res["dram_bytes_per_launch"] = rd + wr
    return res


def main():
    tag = sys.argv[1]
    config = sys.argv[sys.argv.index("--config") + 1] if "--config" in sys.argv else "c4"
    os.makedirs(PROF, exist_ok=True)
    ls = launches(tag)
    with open(os.path.join(PROF, f"{ROUND}_{tag}_launches.csv"), "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=list(ls[0].keys()))
        w.writeheader()
        w.writerows(ls)
    fu = full(tag)
    fu["config"] = config
    with open(os.path.join(PROF, f"{ROUND}_{tag}_ncu_full.json"), "w") as f:
        json.dump(fu, f, indent=1)
    sp = os.path.join(PROF, "ncu_summary.json")
    s = json.load(open(sp)) if os.path.exists(sp) else {}
    s[config] = {"tag": tag, "kernel": fu["kernel"], "dram_bytes_per_launch": fu["dram_bytes_per_launch"],
                 "gpu_time_us": fu["metrics"]["gpu__time_duration.sum"]}
    json.dump(s, open(sp, "w"), indent=1)
    for l in ls[:6]:
        print(l)
    print(json.dumps({k: v["value"] for k, v in fu["metrics"].items()}, indent=0))
    print(fu["stall_share"])


if __name__ == "__main__":
    main()
