"""Shared test helpers: run the CUDA path through the C ABI on seeded ttsynth inputs,
and the oracle on the same inputs; compare with north_star's tolerances."""
from __future__ import annotations

import numpy as np

import oracle
import ttsynth

# north_star: relative L2 error <= 1e-5 per UE and max abs error <= 1e-4 * RMS(y)
REL_L2 = 1e-5
MAX_ABS_RMS = 1e-4


def to_c(a) -> np.ndarray:
    a = np.asarray(a)
    return a[..., 0].astype(np.float64) + 1j * a[..., 1].astype(np.float64)


def compare(y_gpu, y_ref, what=""):
    """Per-channel relative L2 and max-abs/RMS; returns the worst of each."""
    yg = to_c(y_gpu) if np.asarray(y_gpu).dtype != np.complex128 else y_gpu
    yr = y_ref
    assert yg.shape == yr.shape, (yg.shape, yr.shape)
    worst_l2, worst_ma = 0.0, 0.0
    for c in range(yr.shape[0]):
        nrm = np.linalg.norm(yr[c])
        rms = nrm / np.sqrt(yr.shape[1]) if yr.shape[1] else 0.0
        err = yg[c] - yr[c]
        l2 = np.linalg.norm(err) / nrm if nrm > 0 else np.linalg.norm(err)
        ma = np.abs(err).max() / rms if rms > 0 else np.abs(err).max()
        worst_l2, worst_ma = max(worst_l2, l2), max(worst_ma, ma)
    assert worst_l2 <= REL_L2, f"{what}: rel L2 {worst_l2:.3e} > {REL_L2}"
    assert worst_ma <= MAX_ABS_RMS, f"{what}: max-abs/RMS {worst_ma:.3e} > {MAX_ABS_RMS}"
    return worst_l2, worst_ma


def bits_equal(a, b) -> bool:
    """Bitwise equality of float32 arrays, treating +0 and -0 as equal."""
    a = np.asarray(a, dtype=np.float32)
    b = np.asarray(b, dtype=np.float32)
    return a.shape == b.shape and bool(np.all((a == b) | (np.isnan(a) & np.isnan(b)))) and \
        bool(np.array_equal(a.view(np.uint32) & 0x7FFFFFFF, b.view(np.uint32) & 0x7FFFFFFF) or np.all(a == b))


class Run:
    """Inputs of one workload slice (global channels [c_lo, c_hi)) generated with one
    ttsynth backend, kept on the host for the oracle."""

    def __init__(self, w: ttsynth.Workload, c_lo: int = 0, c_hi: int | None = None, calls: list[int] | None = None,
                 seed: int = 0):
        self.w = w
        self.c_lo, self.c_hi = c_lo, (w.C if c_hi is None else c_hi)
        self.C = self.c_hi - self.c_lo
        self.calls = calls if calls is not None else [w.n_per_call] * w.calls
        self.N = int(sum(self.calls))
        self.K = (self.N - 1) // w.S + 2
        self.delays = ttsynth.delays(w, self.c_lo, self.c_hi)
        self.gains = ttsynth.snapshots(w, self.c_lo, self.c_hi, self.K)
        self.x = np.concatenate([ttsynth.iq(w, self.c_lo, self.c_hi, i, n) for i, n in enumerate(self.calls)], axis=1) \
            if self.N else np.zeros((self.C, 0, 2), np.float32)
        self.sigma = float(w.sigma)
        self.seed = seed

    def oracle(self, n0: int = 0, N: int | None = None) -> np.ndarray:
        N = self.N - n0 if N is None else N
        return oracle.convolve(self.delays, self.w.S, self.gains, 0, self.x, 0, n0, N, sigma=self.sigma,
                               seed=self.seed, c_offset=self.c_lo)

    def gpu(self, device, calls: list[int] | None = None, host_path: bool = False, cap: int | None = None):
        """Stream the input through the C ABI in `calls` pieces; returns float32 [C][N][2]."""
        import torch

        from paper_2601_08217_b200 import Channel

        calls = self.calls if calls is None else calls
        assert sum(calls) == self.N
        ch = Channel(self.delays, self.w.S, seed=self.seed, snapshot_capacity=cap or self.K, channel_offset=self.c_lo,
                     device=device)
        try:
            ch.load_snapshots(torch.from_numpy(self.gains).to(device), 0)
            out = np.empty((self.C, self.N, 2), np.float32)
            pos = 0
            for n in calls:
                xs = torch.from_numpy(np.ascontiguousarray(self.x[:, pos:pos + n])).to(device)
                if host_path:
                    xh = xs.cpu().pin_memory()
                    yh = torch.empty_like(xh).pin_memory()
                    ch.apply_host(xh, yh, noise_sigma=self.sigma)
                    torch.cuda.current_stream().synchronize()
                    out[:, pos:pos + n] = yh.numpy()
                else:
                    y = ch.apply(xs, noise_sigma=self.sigma)
                    out[:, pos:pos + n] = y.cpu().numpy()
                pos += n
            torch.cuda.synchronize()
            assert ch.t == self.N
        finally:
            ch.close()
        return out
