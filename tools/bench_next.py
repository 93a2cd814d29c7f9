#!/usr/bin/env python
"""Measurement of the NEXT rows on one GPU, one JSON line each.

    python tools/bench_next.py [--steps K] [--warmup W] [--modes aggregate,sparse,links,synth,load]

Workloads (synthetic, built from BASELINE c4: 122.88 Msps, 0.5 ms slots of 61,440
samples, 48 taps in [0, 1024], S = 256):
  aggregate (f1)  the 512 UL channels of c4 summed into one cell per slot
                  (tt_channel_apply_aggregate, G = 512, per-channel outputs not stored)
  sparse    (f2)  c4 (1024 channels, 10 dB) with the top-20 taps per interval
                  ("over 20 channel taps")
  links     (f4)  512 UEs x 3 gNBs = 1536 links reading 3 shared gNB streams, summed per
                  UE (tt_channel_set_input_map + aggregate, G = 3)
  synth     (f3)  Jakes synthesis of one slot's snapshots for c4's 1024 channels
                  (24 paths -> 48 grid taps, M = 32 sinusoids, 240 snapshots per slot)
  load      (a1)  one c4 slot of snapshots loaded from a device buffer into the ring
Device-timed with CUDA events over K steps after W warm-up steps; inputs resident.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402
import ttsynth  # noqa: E402


def timed(fn, steps, warmup, stream):
    import torch

    for i in range(warmup):
        fn(i)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    with bench.ClockSampler(0) as clk:
        ev[0].record(stream)
        for i in range(steps):
            fn(warmup + i)
            ev[i + 1].record(stream)
        torch.cuda.synchronize()
    per = [ev[i].elapsed_time(ev[i + 1]) for i in range(steps)]
    return ev[0].elapsed_time(ev[-1]), per, clk.summary()


def line(mode, metric, value, unit, steps, warmup, ms, per, clk, config, extra=None):
    d = {"mode": mode, "metric": metric, "value": value, "unit": unit, "n_gpus": 1, "steps": steps,
         "warmup": warmup, "ms_per_step": ms, "higher_is_better": True, "dtype": "f32", "data": "synthetic",
         "config": config, "call_ms": {"p50": statistics.median(per), "p99": float(np.percentile(per, 99))},
         "clocks": clk}
    if extra:
        d.update(extra)
    print(json.dumps(d), flush=True)


def fp32_peak(peaks):
    return bench.SM_COUNT_NOMINAL * bench.FP32_LANES_PER_SM * 2 * peaks["sm_max_mhz"] * 1e6


def run_aggregate(args, dev, peaks):
    import torch

    from paper_2601_08217_b200 import Channel

    w = ttsynth.get("c4").scaled(dirs=1)  # the 512 UL channels
    C, n = w.C, w.n_per_call
    steps_total = args.warmup + args.steps + 1
    K = (steps_total * n - 1) // w.S + 2
    P = min(steps_total, max(2, math.ceil(4 * bench.L2_BYTES / (C * n * 8))))
    xs = [ttsynth.iq(w, 0, C, i, backend="torch", device=dev) for i in range(P)]
    agg = torch.empty((1, n, 2), dtype=torch.float32, device=dev)
    ch = Channel(ttsynth.delays(w), w.S, seed=1, snapshot_capacity=K, device=dev)
    ch.load_snapshots(ttsynth.snapshots(w, 0, C, K, backend="torch", device=dev), 0)
    torch.cuda.synchronize()
    el, per, clk = timed(lambda i: ch.apply_aggregate(xs[i % P], C, agg=agg, noise_sigma=w.sigma), args.steps,
                         args.warmup, torch.cuda.current_stream())
    ch.close()
    ms = el / args.steps
    sps = C * n / (ms / 1e3)
    ach = 8.0 * w.L * sps / 1e12
    line("aggregate", "UL channel samples convolved and summed per s (one cell)", sps, "samples/s", args.steps,
         args.warmup, ms, per, clk,
         {"workload": "c4 UL: 512 UL channels -> 1 cell aggregate per 0.5 ms slot (NEXT f1)", "channels": C,
          "group": C, "samples_per_call": n, "taps": w.L, "snapshot_period": w.S, "snr_db": w.snr_db},
         {"roofline": {"bound": "alu", "achieved": ach, "peak": fp32_peak(peaks) / 1e12, "unit": "TFLOP/s",
                       "frac": ach / (fp32_peak(peaks) / 1e12)},
          "realtime_ues": int(sps // w.rate_sps)})


def run_sparse(args, dev, peaks, top_n=20):
    import torch

    from paper_2601_08217_b200 import Channel

    w = ttsynth.get("c4")
    C, n = w.C, w.n_per_call
    steps_total = args.warmup + args.steps + 1
    K = (steps_total * n - 1) // w.S + 2
    P = min(steps_total, max(2, math.ceil(4 * bench.L2_BYTES / (C * n * 8))))
    xs = [ttsynth.iq(w, 0, C, i, backend="torch", device=dev) for i in range(P)]
    y = torch.empty_like(xs[0])
    ch = Channel(ttsynth.delays(w), w.S, seed=1, snapshot_capacity=K, device=dev)
    ch.set_top_n(top_n)
    ch.load_snapshots(ttsynth.snapshots(w, 0, C, K, backend="torch", device=dev), 0)
    torch.cuda.synchronize()
    el, per, clk = timed(lambda i: ch.apply(xs[i % P], out=y, noise_sigma=w.sigma), args.steps, args.warmup,
                         torch.cuda.current_stream())
    ch.close()
    ms = el / args.steps
    sps = C * n / (ms / 1e3)
    ach = 8.0 * top_n * sps / 1e12
    line("sparse", "channel-convolved complex samples/s, top-%d taps" % top_n, sps, "samples/s", args.steps,
         args.warmup, ms, per, clk,
         {"workload": "c4 with the top-%d of 48 taps per snapshot interval (NEXT f2)" % top_n, "channels": C,
          "samples_per_call": n, "taps": w.L, "top_n": top_n, "snapshot_period": w.S, "snr_db": w.snr_db},
         {"roofline": {"bound": "alu", "achieved": ach, "peak": fp32_peak(peaks) / 1e12, "unit": "TFLOP/s",
                       "frac": ach / (fp32_peak(peaks) / 1e12), "flops_per_sample": 8 * top_n},
          "realtime_ues": w.realtime_ues(sps)})


def run_links(args, dev, peaks, B=3):
    import torch

    from paper_2601_08217_b200 import Channel

    base = ttsynth.get("c4")
    w = base.scaled(ues=base.ues * B, dirs=1)  # link (u, b) = channel u*B + b
    C, n = w.C, w.n_per_call
    steps_total = args.warmup + args.steps + 1
    K = (steps_total * n - 1) // w.S + 2
    xs = [ttsynth.iq(w, 0, B, i, backend="torch", device=dev) for i in range(4)]  # the gNB streams
    agg = torch.empty((base.ues, n, 2), dtype=torch.float32, device=dev)
    ch = Channel(ttsynth.delays(w), w.S, seed=1, snapshot_capacity=K, device=dev)
    ch.set_input_map(np.tile(np.arange(B, dtype=np.int32), base.ues), B)
    ch.load_snapshots(ttsynth.snapshots(w, 0, C, K, backend="torch", device=dev), 0)
    torch.cuda.synchronize()
    el, per, clk = timed(lambda i: ch.apply_aggregate(xs[i % 4], B, agg=agg, noise_sigma=w.sigma), args.steps,
                         args.warmup, torch.cuda.current_stream())
    ch.close()
    ms = el / args.steps
    sps = C * n / (ms / 1e3)
    ach = 8.0 * w.L * sps / 1e12
    line("links", "link samples convolved per s (UE received sums over B gNBs)", sps, "samples/s", args.steps,
         args.warmup, ms, per, clk,
         {"workload": "512 UEs x %d gNBs: 1536 links from 3 shared gNB streams, summed per UE (NEXT f4)" % B,
          "links": C, "gnbs": B, "samples_per_call": n, "taps": w.L, "snapshot_period": w.S},
         {"roofline": {"bound": "alu", "achieved": ach, "peak": fp32_peak(peaks) / 1e12, "unit": "TFLOP/s",
                       "frac": ach / (fp32_peak(peaks) / 1e12)},
          "realtime_ues": int((sps / B) // w.rate_sps)})


def run_synth(args, dev, peaks, P=24, M=32):
    import torch

    from paper_2601_08217_b200 import synth_jakes

    w = ttsynth.get("c4")
    C = w.C
    per_slot = w.n_per_call // w.S  # snapshots per 0.5 ms slot
    rng = np.random.default_rng(0)
    tau = np.sort(rng.uniform(0, 1023, (C, P)), axis=1).astype(np.float32)
    pw = np.exp(-3 * tau / 1024).astype(np.float32)
    pw /= pw.sum(axis=1, keepdims=True)
    nu = 194.4 * w.S / w.rate_sps  # 60 km/h at 3.5 GHz

    def step(i):
        synth_jakes(tau, pw, M, nu, seed=3, first_index=i * per_slot, count=per_slot, device=dev)

    el, per, clk = timed(step, args.steps, args.warmup, torch.cuda.current_stream())
    ms = el / args.steps
    terms = C * P * per_slot * M
    line("synth", "Jakes path-snapshots synthesised per s", C * P * per_slot / (ms / 1e3), "path-snapshots/s",
         args.steps, args.warmup, ms, per, clk,
         {"workload": "c4 channels x 24 paths x 240 snapshots per slot, M=32, f_D=194.4 Hz (NEXT f3)",
          "channels": C, "paths": P, "sinusoids": M, "snapshots_per_step": per_slot, "nu": nu},
         {"sinusoid_terms_per_s": terms / (ms / 1e3),
          "note": "includes host path validation, table build and a stream sync per call"})


def run_load(args, dev, peaks):
    """a1: snapshot loading as a streaming user does it — one slot's snapshots (c4: 1024
    channels x 240 snapshots x 48 taps) copied from a device buffer into the ring each
    step (tt_channel_load_snapshots -> tt_load_kernel: tap sort + (g, dg) rows)."""
    import torch

    from paper_2601_08217_b200 import Channel

    w = ttsynth.get("c4")
    C = w.C
    per = w.n_per_call // w.S
    steps_total = args.warmup + args.steps + 2
    g = ttsynth.snapshots(w, 0, C, steps_total * per + 1, backend="torch", device=dev)
    ch = Channel(ttsynth.delays(w), w.S, seed=1, snapshot_capacity=4 * per, device=dev)
    blocks = [g[:, i * per:(i + 1) * per].contiguous() for i in range(steps_total)]
    el, pr, clk = timed(lambda i: ch.load_snapshots(blocks[i], i * per), args.steps, args.warmup,
                        torch.cuda.current_stream())
    ch.close()
    ms = el / args.steps
    nbytes = C * per * w.L * (8 + 16)  # read (g) + write (g, dg) per tap-snapshot
    line("load", "tap-snapshots loaded per s", C * per * w.L / (ms / 1e3), "tap-snapshots/s", args.steps,
         args.warmup, ms, pr, clk,
         {"workload": "c4: one slot of snapshots (1024 x 240 x 48) per step, device source (row a1)",
          "channels": C, "snapshots_per_step": per, "taps": w.L},
         {"roofline": {"bound": "hbm", "achieved": nbytes / (ms / 1e3) / 1e9, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                       "frac": nbytes / (ms / 1e3) / 1e9 / peaks["hbm_gbs"]}})


def run_realtime(args, dev, peaks):
    """Real-time check of the headline metric: the c4 slot loop with the
    UE count the throughput predicts per GPU; real time holds if the p99 per-slot call
    time stays within the 0.5 ms slot."""
    import torch

    from paper_2601_08217_b200 import Channel

    base = ttsynth.get("c4")
    out = []
    for ues in (249, 240, 232, 224):
        w = base.scaled(ues=ues)
        C, n = w.C, w.n_per_call
        steps_total = args.warmup + args.steps + 1
        K = (steps_total * n - 1) // w.S + 2
        P = min(steps_total, max(2, math.ceil(4 * bench.L2_BYTES / (C * n * 8))))
        xs = [ttsynth.iq(w, 0, C, i, backend="torch", device=dev) for i in range(P)]
        y = torch.empty_like(xs[0])
        ch = Channel(ttsynth.delays(w), w.S, seed=1, snapshot_capacity=K, device=dev)
        ch.load_snapshots(ttsynth.snapshots(w, 0, C, K, backend="torch", device=dev), 0)
        torch.cuda.synchronize()
        el, per, clk = timed(lambda i: ch.apply(xs[i % P], out=y, noise_sigma=w.sigma), args.steps, args.warmup,
                             torch.cuda.current_stream())
        ch.close()
        del xs
        torch.cuda.empty_cache()
        out.append({"ues": ues, "p50_ms": statistics.median(per), "p99_ms": float(np.percentile(per, 99)),
                    "slot_ms": 1e3 * n / w.rate_sps, "realtime": float(np.percentile(per, 99)) <= 1e3 * n / w.rate_sps})
    line("realtime", "c4 slot latency at the predicted real-time UE count", out[0]["p99_ms"], "ms", args.steps,
         args.warmup, out[0]["p50_ms"], [o["p50_ms"] for o in out], clk,
         {"workload": "c4 (DL+UL, 48 taps, 10 dB, 61,440-sample slots) with fewer UEs per GPU"},
         {"higher_is_better": False, "per_ue_count": out})


def run_align(args, dev, peaks):
    """Robustness: c4 slot calls whose length is odd (61,441 samples) vs the even 61,440,
    so odd channel rows start 8 B off a 16-B boundary and every other call starts on an
    odd sample (odd-base noise path)."""
    import torch

    from paper_2601_08217_b200 import Channel

    out = []
    for n in (61440, 61441):
        w = ttsynth.get("c4").scaled(n_per_call=n)
        C = w.C
        steps_total = args.warmup + args.steps + 1
        K = (steps_total * n - 1) // w.S + 2
        P = min(steps_total, max(2, math.ceil(4 * bench.L2_BYTES / (C * n * 8))))
        xs = [ttsynth.iq(w, 0, C, i, backend="torch", device=dev) for i in range(P)]
        y = torch.empty_like(xs[0])
        ch = Channel(ttsynth.delays(w), w.S, seed=1, snapshot_capacity=K, device=dev)
        ch.load_snapshots(ttsynth.snapshots(w, 0, C, K, backend="torch", device=dev), 0)
        torch.cuda.synchronize()
        el, per, clk = timed(lambda i: ch.apply(xs[i % P], out=y, noise_sigma=w.sigma), args.steps, args.warmup,
                             torch.cuda.current_stream())
        ch.close()
        del xs
        torch.cuda.empty_cache()
        out.append({"n_per_call": n, "ms_per_call": el / args.steps, "samples_per_s": C * n / (el / args.steps / 1e3)})
    line("align", "c4 slot calls, odd vs even call length", out[1]["samples_per_s"], "samples/s", args.steps,
         args.warmup, out[1]["ms_per_call"], [o["ms_per_call"] for o in out], clk,
         {"workload": "c4 with 61,441-sample calls (odd) vs 61,440 (even)"}, {"per_length": out})


def run_graph(args, dev, peaks):
    """slot loops eager vs captured into one CUDA graph of G calls
    (device-clock mode) for the short-call configs c3 and c1; ms per call, device-timed."""
    import torch

    from paper_2601_08217_b200 import Channel

    G = 10
    res = []
    for name in ("c3", "c1"):
        w = ttsynth.get(name)
        n = w.n_per_call if w.n_per_call % 256 == 0 else (w.n_per_call // 256) * 256
        w = w.scaled(n_per_call=n)
        C = w.C
        reps = max(1, args.steps // G)
        steps_total = (args.warmup + reps + 2) * G * 2 + 1
        K = (steps_total * n - 1) // w.S + 2
        xs = [ttsynth.iq(w, 0, C, i, backend="torch", device=dev) for i in range(G)]
        ys = [torch.empty_like(x) for x in xs]
        ch = Channel(ttsynth.delays(w), w.S, seed=1, snapshot_capacity=K, device=dev)
        ch.load_snapshots(ttsynth.snapshots(w, 0, C, K, backend="torch", device=dev), 0)
        torch.cuda.synchronize()
        st = torch.cuda.current_stream()
        el_e, per_e, clk = timed(lambda i: ch.apply(xs[i % G], out=ys[i % G], noise_sigma=w.sigma), reps * G,
                                 args.warmup * G, st)
        ch.set_device_clock(True)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for k in range(G):
                ch.apply(xs[k], out=ys[k], noise_sigma=w.sigma)
        el_g, per_g, _ = timed(lambda i: g.replay(), reps, args.warmup, st)
        ch.set_device_clock(False)
        ch.close()
        res.append({"config": name, "channels": C, "samples_per_call": n, "calls_per_graph": G,
                    "eager_ms_per_call": el_e / (reps * G), "graph_ms_per_call": el_g / (reps * G),
                    "speedup": (el_e / (reps * G)) / (el_g / (reps * G))})
        del xs, ys
        torch.cuda.empty_cache()
    line("graph", "slot calls per s, eager vs CUDA graph (device clock)", 1e3 / res[0]["graph_ms_per_call"],
         "calls/s", args.steps, args.warmup, res[0]["graph_ms_per_call"], [r["graph_ms_per_call"] for r in res], clk,
         {"workload": "c3 and c1 slot loops, 10 calls per graph"}, {"per_config": res})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--modes", default="aggregate,sparse,links,synth,load")
    args = ap.parse_args()
    import torch

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    peaks = bench._peaks()
    for m in args.modes.split(","):
        {"aggregate": run_aggregate, "sparse": run_sparse, "links": run_links, "synth": run_synth,
         "load": run_load, "realtime": run_realtime, "align": run_align,
         "graph": run_graph}[m](args, dev, peaks)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
