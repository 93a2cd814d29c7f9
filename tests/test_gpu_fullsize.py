"""Parity at BASELINE.json's FULL sizes, in the launch configuration bench.py times
(one handle over every channel, seed 12345, channel_offset 0, snapshots preloaded,
slot-streamed calls with the delay line carried), on sampled output windows the
oracle computes directly from the same float32 inputs: the stream start, every slot
boundary, tile boundaries, windows in the middle and the ragged end, on the first,
last and randomly drawn channels. Inputs are drawn on the device by ttsynth (as the
bench does) and copied to the host for the oracle; no expected value comes from the
CUDA path."""
import numpy as np
import pytest

import oracle
import ttsynth
from harness import MAX_ABS_RMS, REL_L2

pytestmark = pytest.mark.gpu

SEED = 12345
WIN = 1024


def _windows(w, N, calls, rng):
    n = w.n_per_call
    starts = {0, max(0, N - WIN), max(0, N - 3)}
    for s in range(1, calls):
        starts.add(s * n - WIN // 2)
    for t in (4096, 8192, 16384, 4096 * 7):  # tile boundaries of the tiled plans
        if t + WIN // 2 < N:
            starts.add(t - WIN // 2)
    starts.update(int(v) for v in rng.integers(0, max(1, N - WIN), size=3))
    return sorted(s for s in starts if 0 <= s < N)


@pytest.mark.parametrize("name,calls", [
    ("c1", 1), ("c2", 1), ("c3", 3), ("c4", 3),
    ("c5-L1", 1), ("c5-L4", 1), ("c5-L16", 1), ("c5-L64", 1), ("c5-L256", 1),
])
def test_full_size_sampled_windows(cuda_device, name, calls):
    import torch

    from paper_2601_08217_b200 import Channel

    w = ttsynth.get(name)
    C, n = w.C, w.n_per_call
    N = calls * n
    K = (N - 1) // w.S + 2
    d = ttsynth.delays(w)
    g = ttsynth.snapshots(w, 0, C, K, backend="torch", device=cuda_device)
    xs = [ttsynth.iq(w, 0, C, i, backend="torch", device=cuda_device) for i in range(calls)]
    ys = []
    with Channel(d, w.S, seed=SEED, snapshot_capacity=K, channel_offset=0, device=cuda_device) as ch:
        ch.load_snapshots(g, 0)
        for x in xs:
            ys.append(ch.apply(x, noise_sigma=w.sigma))
        torch.cuda.synchronize()
        assert ch.t == N

    rng = np.random.default_rng(hash(name) & 0xFFFF)
    chans = sorted({0, C - 1, *(int(c) for c in rng.integers(0, C, size=2))})
    worst = (0.0, 0.0)
    for c in chans:
        x_c = torch.cat([x[c] for x in xs], dim=0)  # [N][2] on the device
        y_c = torch.cat([y[c] for y in ys], dim=0)
        for n0 in _windows(w, N, calls, rng):
            m = min(WIN, N - n0)
            x0 = max(0, n0 - w.D)
            k_lo, k_hi = n0 // w.S, (n0 + m - 1) // w.S + 1
            xs_h = x_c[x0:n0 + m].cpu().numpy()[None]
            gs_h = g[c, k_lo:k_hi + 1].cpu().numpy()[None]
            ref = oracle.convolve(d[c:c + 1], w.S, gs_h, k_lo, xs_h, x0, n0, m, sigma=w.sigma, seed=SEED,
                                  c_offset=c)[0]
            got = y_c[n0:n0 + m].cpu().numpy().astype(np.float64)
            got = got[:, 0] + 1j * got[:, 1]
            nrm = np.linalg.norm(ref)
            rms = nrm / np.sqrt(m)
            err = got - ref
            rel = np.linalg.norm(err) / nrm
            mabs = np.abs(err).max() / rms
            assert rel <= REL_L2 and mabs <= MAX_ABS_RMS, (name, c, n0, rel, mabs)
            worst = (max(worst[0], rel), max(worst[1], mabs))
    print(f"{name}: {len(chans)} channels, worst rel L2 {worst[0]:.2e}, max-abs/RMS {worst[1]:.2e}")
    del g, xs, ys
    torch.cuda.empty_cache()
