"""Maximum sizes (GPU, through the C ABI): calls of the largest allowed length
(n_samples = 2^30), odd lengths among them (the robust variant), and a stream position
that passes 2^31, 2^32 and 2^33 samples: the 32-bit boundaries of the kernels' per-call
index math, of t / S and t mod S, and of the Philox counter (m = n / 2 passes 2^31 and
2^32, so its high word becomes 1). Outputs are checked against the oracle on windows at
the call boundaries, around those crossings and at the ragged end; the oracle computes
each window from the same float32 inputs (copied back from the device) and the same gain
snapshots.

About 40 GB of device memory (two channels, 16 GB of input and of output per call);
9.7e9 samples per channel in about 4 s."""
import numpy as np
import pytest

import oracle
import ttsynth
from harness import MAX_ABS_RMS, REL_L2

pytestmark = pytest.mark.gpu

N_MAX = 1 << 30
WIN = 512


def test_max_call_length_and_stream_past_2_pow_32(cuda_device):
    import torch

    from paper_2601_08217_b200 import Channel

    # 1 UE x DL/UL, 8 taps in [0, 1000], S = 2^16 (K ~ 82k snapshots), 10 dB AWGN
    w = ttsynth.get("c4").scaled(ues=1, dirs=2, L=8, D=1000, S=1 << 16, snr_db=10.0, n_per_call=N_MAX, calls=9)
    calls = [N_MAX, N_MAX - 77, N_MAX, N_MAX - 3, N_MAX, N_MAX, N_MAX - 1, N_MAX, N_MAX]
    N = sum(calls)
    assert N > (1 << 33) + (1 << 30) // 2
    C = w.C
    K = (N - 1) // w.S + 2
    d = ttsynth.delays(w)
    g = ttsynth.snapshots(w, 0, C, K)  # host, ~40 MB
    seed = 99

    # windows to check (global sample index of their first output)
    starts = {0, N - WIN}
    pos = 0
    for n in calls[:-1]:
        pos += n
        starts.update((pos - WIN // 2, pos - 3))
    for b in (1 << 31, 1 << 32, 1 << 33):
        starts.update((b - WIN // 2, b - 1, b + 4096 - WIN // 2))
    starts = sorted(s for s in starts if 0 <= s <= N - WIN)

    got = {}
    xwin = {}  # per window: the inputs [s - D, s + WIN) of both channels
    with Channel(d, w.S, seed=seed, snapshot_capacity=K, device=cuda_device) as ch:
        ch.load_snapshots(torch.from_numpy(g).to(cuda_device), 0)
        y_flat = torch.empty(C * N_MAX * 2, dtype=torch.float32, device=cuda_device)
        t0 = 0
        for i, n in enumerate(calls):
            x = ttsynth.iq(w, 0, C, i, n, backend="torch", device=cuda_device)
            y = y_flat[:C * n * 2].view(C, n, 2)
            ch.apply(x, out=y, noise_sigma=w.sigma)
            torch.cuda.synchronize()
            for s in starts:
                lo, hi = s - w.D, s + WIN
                if hi <= t0 or lo >= t0 + n:
                    continue
                # the outputs in this call
                a, b = max(s, t0), min(s + WIN, t0 + n)
                if a < b:
                    got.setdefault(s, np.zeros((C, WIN, 2), np.float32))[:, a - s:b - s] = \
                        y[:, a - t0:b - t0].cpu().numpy()
                # the inputs in this call
                a, b = max(lo, t0), min(hi, t0 + n)
                if a < b:
                    xwin.setdefault(s, np.zeros((C, hi - max(lo, 0), 2), np.float32))[:, a - max(lo, 0):b - max(lo, 0)] = \
                        x[:, a - t0:b - t0].cpu().numpy()
            del x, y
            t0 += n
        assert ch.t == N
        del y_flat
    torch.cuda.empty_cache()

    worst = (0.0, 0.0)
    for s in starts:
        x0 = max(0, s - w.D)
        k_lo, k_hi = s // w.S, (s + WIN - 1) // w.S + 1
        ref = oracle.convolve(d, w.S, g[:, k_lo:k_hi + 1], k_lo, xwin[s], x0, s, WIN, sigma=w.sigma, seed=seed)
        yg = got[s][..., 0].astype(np.float64) + 1j * got[s][..., 1]
        for c in range(C):
            nrm = np.linalg.norm(ref[c])
            err = yg[c] - ref[c]
            rel = np.linalg.norm(err) / nrm
            mabs = np.abs(err).max() / (nrm / np.sqrt(WIN))
            assert rel <= REL_L2 and mabs <= MAX_ABS_RMS, (s, c, rel, mabs)
            worst = (max(worst[0], rel), max(worst[1], mabs))
    print(f"max sizes: {len(starts)} windows up to t = {N}, worst rel L2 {worst[0]:.2e}, max-abs/RMS {worst[1]:.2e}")


def test_many_channels_with_global_ids_past_2_pow_32(cuda_device):
    """65,536 channels in one handle whose global ids (channel_offset + c) wrap past 2^32:
    the noise key is the global id mod 2^32 on both sides (docs/tt-normal-v1.md §1), and
    the per-channel offsets into the ring, history and buffers are 64-bit. Two streamed
    calls; sampled channels (first, around the wrap, last, random) vs the oracle."""
    import torch

    from paper_2601_08217_b200 import Channel

    rng = np.random.default_rng(2026)
    C, L, D, S = 1 << 16, 16, 200, 256
    calls = [2048, 1536]
    N = sum(calls)
    K = (N - 1) // S + 2
    off = (1 << 32) - 30_000
    d = np.concatenate([np.zeros((C, 1), np.int64), np.sort(rng.integers(1, D + 1, size=(C, L - 1)), axis=1)],
                       axis=1).astype(np.int32)
    g = (rng.standard_normal((C, K, L, 2)) * np.sqrt(0.5 / L)).astype(np.float32)
    x = (rng.standard_normal((C, N, 2)) * np.sqrt(0.5)).astype(np.float32)
    sigma = 0.1
    ys = []
    with Channel(d, S, seed=5, snapshot_capacity=K, channel_offset=off, device=cuda_device) as ch:
        ch.load_snapshots(torch.from_numpy(g).to(cuda_device), 0)
        pos = 0
        for n in calls:
            ys.append(ch.apply(torch.from_numpy(np.ascontiguousarray(x[:, pos:pos + n])).to(cuda_device),
                               noise_sigma=sigma).cpu().numpy())
            pos += n
        torch.cuda.synchronize()
    y = np.concatenate(ys, axis=1)
    wrap = (1 << 32) - off
    chans = sorted({0, 1, wrap - 2, wrap - 1, wrap, wrap + 1, C - 1, *(int(c) for c in rng.integers(0, C, 4))})
    for c in chans:
        ref = oracle.convolve(d[c:c + 1], S, g[c:c + 1], 0, x[c:c + 1], 0, 0, N, sigma=sigma, seed=5,
                              c_offset=off + c)[0]
        yg = y[c, :, 0].astype(np.float64) + 1j * y[c, :, 1]
        nrm = np.linalg.norm(ref)
        err = yg - ref
        assert np.linalg.norm(err) / nrm <= REL_L2, c
        assert np.abs(err).max() / (nrm / np.sqrt(N)) <= MAX_ABS_RMS, c
