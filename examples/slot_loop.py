#!/usr/bin/env python
"""A Tiny-Twin slot loop on one GPU: for every 0.5 ms slot, synthesise the next slot's
channel snapshots on the GPU (Jakes, NEXT f3), load them into the ring (a1), and
convolve the slot's IQ of every UE's DL and UL channel with noise (a2-a6).

    python examples/slot_loop.py [--ues 512] [--slots 50]

Workload shape follows BASELINE c4: 122.88 Msps, 61,440-sample slots, 24 paths with an
exponential power-delay profile over [0, 1024) samples (-> 48 grid taps), S = 256,
10 dB SNR, 60 km/h at 3.5 GHz. Inputs are synthetic; prints the time per slot of each
stage and the real-time factor (slot time / wall time per slot).
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_08217_b200 import Channel, synth_jakes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ues", type=int, default=512)
    ap.add_argument("--slots", type=int, default=50)
    ap.add_argument("--paths", type=int, default=24)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    rate, n, S, P, M = 122.88e6, 61_440, 256, args.paths, 32
    C = 2 * args.ues                     # channel 2u = DL, 2u + 1 = UL
    per = n // S                         # snapshots per slot
    nu = 194.4 * S / rate                # Doppler per snapshot period
    sigma = 10 ** (-10 / 20)             # 10 dB SNR at unit signal power
    rng = np.random.default_rng(1)
    tau = np.sort(rng.uniform(0, 1023, (C, P)), axis=1).astype(np.float32)
    pw = np.exp(-3 * tau / 1024).astype(np.float32)
    pw /= pw.sum(axis=1, keepdims=True)

    # snapshots 0 .. per (slot 0 needs its intervals' both ends)
    delays, g0 = synth_jakes(tau, pw, M, nu, seed=7, first_index=0, count=per + 1, device=dev)
    ch = Channel(delays, S, seed=11, snapshot_capacity=2 * per + 2, device=dev)
    ch.load_snapshots(g0, 0)
    xs = [torch.randn((C, n, 2), device=dev) * np.float32(np.sqrt(0.5)) for _ in range(2)]
    ys = [torch.empty_like(x) for x in xs]
    ev = {k: [torch.cuda.Event(enable_timing=True) for _ in range(args.slots + 1)] for k in ("synth", "load", "apply")}
    t_synth = t_load = t_apply = 0.0
    total0, total1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    total0.record()
    for s in range(args.slots):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        e[0].record()
        # the next slot's snapshots: (s + 1) per + 1 .. (s + 2) per
        _, g = synth_jakes(tau, pw, M, nu, seed=7, first_index=(s + 1) * per + 1, count=per, device=dev)
        e[1].record()
        ch.load_snapshots(g, (s + 1) * per + 1)
        e[2].record()
        ch.apply(xs[s % 2], out=ys[s % 2], noise_sigma=sigma)
        e[3].record()
        torch.cuda.synchronize()
        t_synth += e[0].elapsed_time(e[1])
        t_load += e[1].elapsed_time(e[2])
        t_apply += e[2].elapsed_time(e[3])
    total1.record()
    torch.cuda.synchronize()
    wall = total0.elapsed_time(total1) / args.slots
    k = args.slots
    print(f"{args.ues} UEs ({C} channels), {P} paths -> {delays.shape[1]} taps, {k} slots of {n} samples")
    print(f"per slot: synth {t_synth / k:.3f} ms, load {t_load / k:.3f} ms, apply {t_apply / k:.3f} ms, "
          f"wall {wall:.3f} ms; real-time factor {1e3 * n / rate / wall:.2f}")
    ch.close()


if __name__ == "__main__":
    main()
