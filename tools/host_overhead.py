#!/usr/bin/env python
"""Host-side cost of one tt_channel_apply through the Python binding: wall time per
call of a tiny slot loop, GPU work negligible (1 channel x 256 samples)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import ttsynth  # noqa: E402
from paper_2601_08217_b200 import Channel, _lib  # noqa: E402

dev = torch.device("cuda", 0)
w = ttsynth.get("c1").scaled(n_per_call=256, calls=20_000)
K = (w.calls * 256) // w.S + 3
ch = Channel(ttsynth.delays(w), w.S, seed=1, snapshot_capacity=K, device=dev)
ch.load_snapshots(ttsynth.snapshots(w, 0, w.C, K, backend="torch", device=dev), 0)
x = ttsynth.iq(w, 0, w.C, 0, backend="torch", device=dev)
y = torch.empty_like(x)
res = {}
for label, fn in (
    ("Channel.apply", lambda: ch.apply(x, out=y)),
    ("_lib.tt_channel_apply (stream given)", lambda s=torch.cuda.current_stream().cuda_stream: _lib.tt_channel_apply(
        ch.handle, x.data_ptr(), y.data_ptr(), 256, 0.0, s)),
):
    for _ in range(200):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5000):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    res[label] = (t1 - t0) / 5000 * 1e6
print(json.dumps({"us_per_call_host": res}))
