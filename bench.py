#!/usr/bin/env python
"""Benchmark of the Tiny-Twin channel convolution hot path (BASELINE.json metric:
channel-convolved complex samples/s for the whole box, real-time UE count, %
roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl reference]

Workload (default c4, BASELINE.json configs[3]: 512 UEs x DL/UL, 48 taps in
[0, 1024], snapshots every 256 samples, 10 dB AWGN, 0.5 ms slots of 61,440
samples at 122.88 Msps, "sharded across 1/2/4/8 GPUs"). One step = one slot: one
`tt_channel_apply` over every channel this rank owns, with the delay line carried
from the previous slot. UEs are sharded in contiguous blocks over ranks (no
collective on the data path; NCCL only for the barrier and the max-over-ranks
timing). Inputs are synthetic (ttsynth) and resident in HBM before timing; a
rotating pool of distinct slot buffers totalling >= 4x L2 is cycled so no step's
input is L2-resident. See DESIGN.md §6 for the roofline and metric definitions.

Under torchrun every rank runs its shard; rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import ttsynth  # noqa: E402

L2_BYTES = 126 * 1024 * 1024
SM_COUNT_NOMINAL = 148
FP32_LANES_PER_SM = 128  # FFMA lanes per SM per clock (2 flop each)


def _peaks():
    p = {"hbm_gbs": 6549.8, "sm_max_mhz": 1965.0, "source": "fallback"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        p.update(hbm_gbs=float(m["hbm_gbs"]), sm_max_mhz=float(m.get("sm_max_mhz", 1965.0)), source="measured")
    except Exception:
        pass
    return p


class ClockSampler:
    """Samples SM clock and throttle reasons via NVML during the timed region."""

    BAD = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
           "hw_power_brake_slowdown": 0x80}
    NOTE = {"sw_power_cap": 0x4}

    def __init__(self, index: int, period_s: float = 0.01):
        self.index, self.period = index, period_s
        self.samples, self.reasons, self.power = [], 0, []
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM))
                self.reasons |= int(self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h))
                self.power.append(self._nv.nvmlDeviceGetPowerUsage(self._h) / 1000.0)  # W
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self._nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if self._nv is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        names = [k for k, v in {**self.BAD, **self.NOTE}.items() if self.reasons & v]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": names, "samples": len(self.samples),
                "power_w_median": statistics.median(self.power) if self.power else None}


def _dist():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def roofline(w: ttsynth.Workload, samples: int, kernel_s: float, peaks: dict, traffic):
    """NS roofline: min(HBM / 16 B per sample, FP32 / 8L flop per sample) per GPU."""
    fp32 = SM_COUNT_NOMINAL * FP32_LANES_PER_SM * 2 * peaks["sm_max_mhz"] * 1e6  # flop/s
    hbm = peaks["hbm_gbs"] * 1e9                                                # B/s
    hbm_rate, alu_rate = hbm / 16.0, fp32 / (8.0 * w.L)
    if alu_rate < hbm_rate:
        achieved = 8.0 * w.L * samples / kernel_s / 1e12
        rl = {"bound": "alu", "achieved": achieved, "peak": fp32 / 1e12, "unit": "TFLOP/s"}
    else:
        achieved = 16.0 * samples / kernel_s / 1e9
        rl = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s"}
    rl["frac"] = rl["achieved"] / rl["peak"]
    rl["traffic"] = traffic
    rl["peak_source"] = peaks["source"] + (" (FP32 peak = 148 SM x 128 lanes x 2 x sm_max_mhz)"
                                           if rl["bound"] == "alu" else " (MEASURED_PEAKS.json hbm_gbs)")
    rl["ns_samples_per_s_per_gpu"] = min(hbm_rate, alu_rate)
    return rl


def _ceilings(w, peaks, achieved_sps):
    f = peaks["sm_max_mhz"] * 1e6
    interp = SM_COUNT_NOMINAL * FP32_LANES_PER_SM * f / (6.0 * w.L)   # samples/s
    smem = SM_COUNT_NOMINAL * 16.0 * f / w.L                           # 16 output-taps/clk/SM
    hbm = peaks["hbm_gbs"] * 1e9 / (16.0 + 16.0 * w.L / w.S)          # incl. the gain stream
    lim = min(interp, smem, hbm)
    return {"interp_fp32_sps": interp, "smem_operands_sps": smem, "hbm_with_gains_sps": hbm,
            "frac_of_min": achieved_sps / lim}


def _traffic(config: str):
    """dram read+write bytes per launch from the committed ncu --set full summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            s = json.load(f)
        return s.get(config, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(w: ttsynth.Workload, target_s: float = 10.0):
    """The oracle (as it stands) on this host's cores, on a bounded sample of the
    workload: whole slots of the first channels, grown until ~target_s of wall time."""
    import oracle

    cores = len(os.sched_getaffinity(0))
    n = w.n_per_call
    # probe: one slot of a few channels -> rate; then size (channels, consecutive slots)
    # for ~target_s of oracle work on this workload
    c0 = min(w.C, max(1, cores))
    K = (n - 1) // w.S + 2
    pd, pg, px = ttsynth.delays(w, 0, c0), ttsynth.snapshots(w, 0, c0, K), ttsynth.iq(w, 0, c0, 0)
    best = float("inf")
    for _ in range(2):  # the first call also pays library load / thread-pool start
        t0 = time.perf_counter()
        oracle.convolve(pd, w.S, pg, 0, px, 0, 0, n, sigma=w.sigma, seed=0)
        best = min(best, time.perf_counter() - t0)
    rate = c0 * n / max(best, 1e-4)
    want = rate * target_s
    c = int(min(w.C, max(1, want // n)))
    slots = int(min(w.calls, max(1, want // (c * n))))
    N = slots * n
    K = (N - 1) // w.S + 2
    d = ttsynth.delays(w, 0, c)
    g = ttsynth.snapshots(w, 0, c, K)
    x = np.concatenate([ttsynth.iq(w, 0, c, i) for i in range(slots)], axis=1)
    t0 = time.perf_counter()
    oracle.convolve(d, w.S, g, 0, x, 0, 0, N, sigma=w.sigma, seed=0)
    elapsed = time.perf_counter() - t0
    done = c * N
    return {"value": done / elapsed, "unit": "samples/s", "cores": cores, "kind": "oracle", "cpu": _cpu_model(),
            "sample": f"{c} of {w.C} channels x {slots} consecutive slots of {n} samples of {w.name} "
                      f"({done} samples, {elapsed:.2f} s wall, double precision, OpenMP over {cores} threads)"}


def run_reference(args, w):
    """--impl reference: the oracle timed as the reference arm, rank 0 only."""
    rank, world, _ = _dist()
    if rank != 0:
        return
    import oracle

    cores = len(os.sched_getaffinity(0))
    # each step: one slot of a bounded channel sample, sized for ~1 s of oracle work
    n = w.n_per_call
    K = (n - 1) // w.S + 2
    probe = min(w.C, max(1, cores))
    d = ttsynth.delays(w, 0, probe)
    g = ttsynth.snapshots(w, 0, probe, K)
    x = ttsynth.iq(w, 0, probe, 0)
    oracle.convolve(d, w.S, g, 0, x, 0, 0, n, sigma=w.sigma)  # library load / thread start
    t0 = time.perf_counter()
    oracle.convolve(d, w.S, g, 0, x, 0, 0, n, sigma=w.sigma)
    per_ch = (time.perf_counter() - t0) / probe
    c = int(max(1, min(w.C, 1.0 / max(per_ch, 1e-6))))
    d = ttsynth.delays(w, 0, c)
    g = ttsynth.snapshots(w, 0, c, K)
    x = ttsynth.iq(w, 0, c, 0)
    for _ in range(args.warmup):
        oracle.convolve(d[:c], w.S, g[:c], 0, x[:c], 0, 0, n, sigma=w.sigma)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.convolve(d[:c], w.S, g[:c], 0, x[:c], 0, 0, n, sigma=w.sigma)
        ts.append(time.perf_counter() - t0)
    tot = sum(ts)
    val = c * n * args.steps / tot
    line = {
        "impl": "reference", "metric": "channel-convolved complex samples/s (whole box)", "value": val,
        "unit": "samples/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": _config(w, world),
        "cpu_baseline": {"value": val, "unit": "samples/s", "cores": cores, "kind": "oracle", "cpu": _cpu_model(),
                         "sample": f"{c} of {w.C} channels x 1 slot of {n} samples per step"},
        "e2e": {"value": val, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "realtime_ues": w.realtime_ues(val),
    }
    print(json.dumps(line), flush=True)


def _config(w, world):
    return {"workload": f"BASELINE configs {w.name}", "ues": w.ues, "channels": w.C,
            "channels_per_ue": w.dirs, "samples_per_call": w.n_per_call, "taps": w.L, "max_delay": w.D,
            "snapshot_period": w.S, "snr_db": w.snr_db, "sample_rate_sps": w.rate_sps,
            "parallelism": f"ue-shard x{world}",
            "l2": "rotating pool of distinct slot inputs, >= 4x L2 per rank (inputs not L2-resident)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sigma", type=float, default=None, help="override the config's noise sigma (experiments)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: >= 3 warm-up steps
    w = ttsynth.get(args.config)
    if args.impl == "reference":
        run_reference(args, w)
        return

    import torch

    from paper_2601_08217_b200 import Channel, _lib, shard

    rank, world, local = shard.env()
    if world != args.gpus and rank == 0:
        print(f"note: --gpus {args.gpus} but WORLD_SIZE {world}; using WORLD_SIZE", file=sys.stderr)
    # TT_BENCH_ONE_GPU=1 (tests only): every rank on cuda:0 with a gloo group, to exercise
    # the sharded multi-rank path on a one-GPU box (the ranks' kernels are independent)
    one_gpu = os.environ.get("TT_BENCH_ONE_GPU") == "1"
    local_dev = 0 if one_gpu else local
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    pg = shard.init("gloo" if one_gpu else "nccl", dev)
    red_dev = torch.device("cpu") if one_gpu else dev

    # ---- this rank's shard (contiguous UE block; DL/UL of a UE stay together) ----------
    c_lo, c_hi = shard.ue_block(w.ues, w.dirs, rank, world)
    assert (c_lo, c_hi) == ttsynth.shard_ues(w, rank, world)
    C, n = c_hi - c_lo, w.n_per_call
    steps_total = args.warmup + args.steps + max(args.e2e_steps, 0) + 1
    # streaming configs (c3, c4: many slots) carry the delay line from slot to slot; a
    # one-call config (c1, c2, c5) repeats its single call, the stream reset (t = 0, zero
    # delay line) inside each step
    one_shot = w.calls == 1
    # a streaming config runs its `calls` slots (c4: 100 slots = 50 ms of air time) and then
    # starts over (stream reset: t = 0, zero delay line; no device work), so the snapshots
    # preloaded for it cover at most `calls` slots however long the run
    slots = 1 if one_shot else min(steps_total, w.calls)
    K = (slots * n - 1) // w.S + 2
    delays = ttsynth.delays(w, c_lo, c_hi)
    gains = ttsynth.snapshots(w, c_lo, c_hi, K, backend="torch", device=dev)
    slot_bytes = C * n * 8
    P = max(2, math.ceil(4 * L2_BYTES / max(slot_bytes, 1)))
    P = min(P, steps_total)
    xs = [ttsynth.iq(w, c_lo, c_hi, i, backend="torch", device=dev) for i in range(P)]
    y = torch.empty_like(xs[0])
    ch = Channel(delays, w.S, seed=12345, snapshot_capacity=K, channel_offset=c_lo, device=dev)
    ch.load_snapshots(gains, 0)
    del gains
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    sigma = w.sigma if args.sigma is None else args.sigma

    # ---- device-resident timed region ----------------------------------------------
    slot = [0]  # slots applied since the last stream reset

    def start_slot():
        if slot[0] == slots:
            ch.reset()
            slot[0] = 0
        slot[0] += 1

    def step(xin):
        start_slot()
        ch.apply(xin, out=y, noise_sigma=sigma)

    for i in range(args.warmup):
        step(xs[i % P])
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    shard.barrier(pg)
    torch.cuda.synchronize()
    with ClockSampler(local_dev) as clk:
        ev[0].record(stream)
        for i in range(args.steps):
            step(xs[(args.warmup + i) % P])
            ev[i + 1].record(stream)
        torch.cuda.synchronize()
    shard.barrier(pg)
    per_step = [ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps)]  # ms, one launch each
    elapsed_max = shard.max_over_ranks(ev[0].elapsed_time(ev[-1]), red_dev, pg)
    samples_all = shard.sum_over_ranks(C * n * args.steps, red_dev, pg)  # units all ranks processed
    value = samples_all / (elapsed_max / 1e3)
    kernel_s = statistics.mean(per_step) / 1e3

    # ---- end-to-end through the C ABI with host buffers (H2D + D2H inside) -----------
    e2e = None
    if args.e2e_steps > 0:
        xh = [xs[i % P].cpu().pin_memory() for i in range(min(P, 2))]
        yh = torch.empty_like(xh[0]).pin_memory()
        start_slot()
        ch.apply_host(xh[0], yh, noise_sigma=sigma)  # staging allocation + warm-up
        torch.cuda.synchronize()
        shard.barrier(pg)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(args.e2e_steps):
            start_slot()
            ch.apply_host(xh[i % len(xh)], yh, noise_sigma=sigma)
        e1.record(stream)
        torch.cuda.synchronize()
        te = shard.max_over_ranks(e0.elapsed_time(e1), red_dev, pg)
        e2e = {"value": shard.sum_over_ranks(C * n * args.e2e_steps, red_dev, pg) / (te / 1e3), "unit": "samples/s",
               "h2d_bytes_per_step": slot_bytes, "d2h_bytes_per_step": slot_bytes,
               "steps": args.e2e_steps, "api": "tt_channel_apply_host (pinned host buffers)"}
    info = ch.info()
    ch.close()

    if rank == 0:
        peaks = _peaks()
        rl = roofline(w, C * n, kernel_s, peaks, _traffic(w.name))
        line = {
            "metric": "channel-convolved complex samples/s (whole box)",
            "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": elapsed_max / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": _config(w, world),
            "roofline": rl,
            "realtime_ues": w.realtime_ues(value),
            "ns_fraction_box": value / (world * rl["ns_samples_per_s_per_gpu"]),
            # design ceilings below NS, per GPU: exact per-sample
            # interpolation (6 FMA lanes per output-tap instead of 4) and one 8-B shared-
            # memory operand read per output-tap (128 B/clk/SM)
            "ceilings": _ceilings(w, peaks, C * n / kernel_s),
            "call_ms": {"p50": statistics.median(per_step), "p99": float(np.percentile(per_step, 99)),
                        "slot_ms": 1e3 * n / w.rate_sps},
            "gpu_launches": args.steps * int(info.launches_per_apply),
            "plan": {"kernel": _lib.KERNELS.get(int(info.kernel), "?"),
                     "outputs_per_thread": int(info.outputs_per_thread)},
            "clocks": clk.summary(),
            "e2e": e2e,
        }
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_baseline(w)
        elif not args.no_cpu_baseline:
            line["cpu_baseline"] = {"value": None, "unit": "samples/s", "cores": len(os.sched_getaffinity(0)),
                                    "kind": "oracle", "sample": "reported at N=1 only"}
        print(json.dumps(line), flush=True)
    if pg:
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
