"""Seeded synthetic workloads for the Tiny-Twin channel convolution.

This module is the ONE thing the oracle side (``oracle/``, ``tests/``) and the CUDA
side (``paper_2601_08217_b200``, ``bench.py``) share: it draws inputs (delays,
power-delay profiles, Rayleigh gain snapshots, IQ streams) and holds **none** of
the method's arithmetic (no interpolation, no convolution, no noise transform).

The five presets are BASELINE.json ``configs`` c1..c5 (recipe and readings:
DESIGN.md §4, SURVEY.md §8.3 readings 11-16). The paper's own traces (3GPP+Jakes,
Sionna ray tracing, ARGOS measurements; §IV) are not available; these
synthetic draws stand in for them.

Determinism: every draw is keyed by (master seed, kind, GLOBAL channel or UE id,
call index), so any sharding of UEs over ranks, and any backend call order,
reproduces the same values for the same backend ("numpy" on the CPU, "torch" on a
torch device).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional, Sequence

import numpy as np

KIND_DELAY, KIND_SNAP, KIND_X = 1, 2, 3


@dataclasses.dataclass(frozen=True)
class Workload:
    name: str
    ues: int                 # UEs
    dirs: int                # channel streams per UE (1, or 2 = DL + UL; c = dirs*u + dir)
    n_per_call: int          # samples per channel per apply call
    calls: int               # apply calls (slots)
    L: int                   # taps
    D: int                   # max delay (delays drawn from [0, D])
    S: int                   # snapshot period (samples)
    snr_db: Optional[float]  # None = no noise
    rate_sps: float          # sample rate (for the real-time UE count)
    seed: int                # master seed
    fixed_delays: Optional[Sequence[int]] = None
    fixed_pdp: Optional[Sequence[float]] = None

    @property
    def C(self) -> int:
        return self.ues * self.dirs

    @property
    def total_per_channel(self) -> int:
        return self.n_per_call * self.calls

    @property
    def total_samples(self) -> int:
        return self.C * self.total_per_channel

    @property
    def sigma(self) -> float:
        """Complex noise std: sigma^2 = 10^(-SNR/10) x nominal signal power sum(p)E|x|^2 = 1."""
        return 0.0 if self.snr_db is None else math.sqrt(10.0 ** (-self.snr_db / 10.0))

    @property
    def K_total(self) -> int:
        """Snapshots needed for the whole run: k = 0 .. floor((N-1)/S) + 1."""
        return (self.total_per_channel - 1) // self.S + 2

    def scaled(self, **kw) -> "Workload":
        return dataclasses.replace(self, **kw)

    def realtime_ues(self, samples_per_s: float) -> int:
        return int(samples_per_s // (self.rate_sps * self.dirs))


PRESETS = {
    # c1: 1 UE, one 10 ms frame at 30.72 Msps, 4 taps {0,3,7,12}, PDP {.5,.25,.15,.10}, S=2048, no noise, seed 0
    "c1": Workload("c1", 1, 1, 307_200, 1, 4, 12, 2048, None, 30.72e6, 0, (0, 3, 7, 12), (0.5, 0.25, 0.15, 0.10)),
    # c2: 4 UEs, 1 s at 30.72 Msps, 23 taps in [0,300], exp PDP, S=1024, 20 dB
    "c2": Workload("c2", 4, 1, 30_720_000, 1, 23, 300, 1024, 20.0, 30.72e6, 1),
    # c3: 64 UEs x DL/UL, 61.44 Msps, 0.5 ms slots (30,720) x 200, 23 taps in [0,600], S=512, 15 dB
    "c3": Workload("c3", 64, 2, 30_720, 200, 23, 600, 512, 15.0, 61.44e6, 2),
    # c4: 512 UEs x DL/UL, 122.88 Msps, 100 slots of 61,440, 48 taps in [0,1024], S=256, 10 dB
    "c4": Workload("c4", 512, 2, 61_440, 100, 48, 1024, 256, 10.0, 122.88e6, 3),
}
for _L in (1, 4, 16, 64, 256):
    # c5: 1024 UEs x 1,048,576 samples, delays in [0,4L], S=128, no noise; rate assumed 122.88 Msps (R16)
    PRESETS[f"c5-L{_L}"] = Workload(f"c5-L{_L}", 1024, 1, 1_048_576, 1, _L, 4 * _L, 128, None, 122.88e6, 4)
for _L in (8, 12, 23, 32):
    # extra points of the same sweep that place the HBM / shared-memory knee (SURVEY §8.4
    # "Crossover (c5)"); not BASELINE configs
    PRESETS[f"c5-L{_L}"] = Workload(f"c5-L{_L}", 1024, 1, 1_048_576, 1, _L, 4 * _L, 128, None, 122.88e6, 4)


def get(name: str) -> Workload:
    return PRESETS[name]


def _seed_words(w: Workload, kind: int, ident: int, sub: int = 0) -> np.random.SeedSequence:
    return np.random.SeedSequence([w.seed, kind, ident, sub])


def _torch_seed(w: Workload, kind: int, ident: int, sub: int = 0) -> int:
    return int(_seed_words(w, kind, ident, sub).generate_state(1, dtype=np.uint64)[0] & ((1 << 63) - 1))


def ue_delays(w: Workload, ue: int) -> np.ndarray:
    """Integer delays of UE `ue` (shared by its DL and UL, R11): d_0 = 0 and
    d_1..d_{L-1} a sorted draw without replacement from {1..D} (R13)."""
    if w.fixed_delays is not None:
        return np.asarray(w.fixed_delays, dtype=np.int32)
    if w.L == 1:
        return np.zeros(1, dtype=np.int32)
    rng = np.random.Generator(np.random.PCG64(_seed_words(w, KIND_DELAY, ue)))
    rest = np.sort(rng.choice(np.arange(1, w.D + 1), size=w.L - 1, replace=False))
    return np.concatenate([[0], rest]).astype(np.int32)


def delays(w: Workload, c_lo: int = 0, c_hi: Optional[int] = None) -> np.ndarray:
    """[c_hi - c_lo][L] int32 delays for GLOBAL channels c_lo..c_hi-1."""
    c_hi = w.C if c_hi is None else c_hi
    if c_hi <= c_lo:
        return np.zeros((0, w.L), dtype=np.int32)
    return np.stack([ue_delays(w, c // w.dirs) for c in range(c_lo, c_hi)]).astype(np.int32)


def pdp(w: Workload, d: np.ndarray) -> np.ndarray:
    """Power-delay profile p_l for delays d (last axis): exponential p_l ∝ exp(-3 d_l / D),
    normalised to sum 1 (R14); c1 uses its explicit profile."""
    if w.fixed_pdp is not None:
        return np.broadcast_to(np.asarray(w.fixed_pdp, dtype=np.float64), d.shape).copy()
    p = np.exp(-3.0 * d.astype(np.float64) / max(w.D, 1))
    return p / p.sum(axis=-1, keepdims=True)


def snapshots(w: Workload, c_lo: int, c_hi: int, K: int, backend: str = "numpy", device=None):
    """Rayleigh gain snapshots g[c][k][l] = sqrt(p_l/2)(a + ib), a, b ~ N(0,1) iid over
    (channel, k, tap) (R12), for GLOBAL channels c_lo..c_hi-1 and k = 0..K-1.
    Returns float32 [C][K][L][2] (numpy array or torch tensor on `device`)."""
    d = delays(w, c_lo, c_hi)
    amp = np.sqrt(pdp(w, d) / 2.0).astype(np.float32)  # [C][L]
    if backend == "numpy":
        out = np.empty((c_hi - c_lo, K, w.L, 2), dtype=np.float32)
        for i, c in enumerate(range(c_lo, c_hi)):
            rng = np.random.Generator(np.random.PCG64(_seed_words(w, KIND_SNAP, c, K)))
            out[i] = rng.standard_normal((K, w.L, 2), dtype=np.float32)
        out *= amp[:, None, :, None]
        return out
    import torch
    out = torch.empty((c_hi - c_lo, K, w.L, 2), dtype=torch.float32, device=device)
    gen = torch.Generator(device=device)
    for i, c in enumerate(range(c_lo, c_hi)):
        gen.manual_seed(_torch_seed(w, KIND_SNAP, c, K))
        torch.randn((K, w.L, 2), generator=gen, out=out[i])
    out *= torch.from_numpy(amp).to(device)[:, None, :, None]
    return out


def iq(w: Workload, c_lo: int, c_hi: int, call: int, n: Optional[int] = None, backend: str = "numpy",
       device=None):
    """IQ input x ~ CN(0,1) (each component N(0, 1/2)) for GLOBAL channels c_lo..c_hi-1 and
    apply call `call`: float32 [C][n][2], interleaved (re, im)."""
    n = w.n_per_call if n is None else n
    s = np.float32(math.sqrt(0.5))
    if backend == "numpy":
        out = np.empty((c_hi - c_lo, n, 2), dtype=np.float32)
        for i, c in enumerate(range(c_lo, c_hi)):
            rng = np.random.Generator(np.random.PCG64(_seed_words(w, KIND_X, c, call * 1_000_003 + n)))
            out[i] = rng.standard_normal((n, 2), dtype=np.float32)
        out *= s
        return out
    import torch
    out = torch.empty((c_hi - c_lo, n, 2), dtype=torch.float32, device=device)
    gen = torch.Generator(device=device)
    for i, c in enumerate(range(c_lo, c_hi)):
        gen.manual_seed(_torch_seed(w, KIND_X, c, call * 1_000_003 + n))
        torch.randn((n, 2), generator=gen, out=out[i])
    out *= float(s)
    return out


def shard_ues(w: Workload, rank: int, world: int) -> tuple[int, int]:
    """Contiguous UE block of `rank` (both directions of a UE stay on one rank);
    returns the GLOBAL channel range [c_lo, c_hi)."""
    u_lo = rank * w.ues // world
    u_hi = (rank + 1) * w.ues // world
    return u_lo * w.dirs, u_hi * w.dirs
