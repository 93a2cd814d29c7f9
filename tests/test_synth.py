"""The seeded input generators (ttsynth): BASELINE.json config recipes, determinism
per global channel, and shard independence (any UE sharding reproduces the same
inputs)."""
import numpy as np
import pytest

import ttsynth


def test_presets_match_baseline_configs():
    c1, c2, c3, c4 = (ttsynth.get(k) for k in ("c1", "c2", "c3", "c4"))
    assert (c1.C, c1.n_per_call, c1.L, c1.S, c1.sigma) == (1, 307_200, 4, 2048, 0.0)
    assert list(ttsynth.delays(c1)[0]) == [0, 3, 7, 12]
    assert np.allclose(ttsynth.pdp(c1, ttsynth.delays(c1))[0], [0.5, 0.25, 0.15, 0.10])
    assert (c2.C, c2.n_per_call, c2.L, c2.D, c2.S) == (4, 30_720_000, 23, 300, 1024)
    assert abs(c2.sigma ** 2 - 1e-2) < 1e-15
    assert (c3.C, c3.n_per_call, c3.calls, c3.L, c3.D, c3.S) == (128, 30_720, 200, 23, 600, 512)
    assert abs(c3.sigma ** 2 - 10 ** -1.5) < 1e-15
    assert (c4.C, c4.n_per_call, c4.calls, c4.L, c4.D, c4.S) == (1024, 61_440, 100, 48, 1024, 256)
    assert abs(c4.sigma ** 2 - 0.1) < 1e-15
    for L in (1, 4, 16, 64, 256):
        c5 = ttsynth.get(f"c5-L{L}")
        assert (c5.C, c5.n_per_call, c5.L, c5.D, c5.S, c5.sigma) == (1024, 1_048_576, L, 4 * L, 128, 0.0)


@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c5-L256", "c5-L1"])
def test_delay_recipe(name):
    w = ttsynth.get(name)
    d = ttsynth.delays(w, 0, min(w.C, 16))
    assert d.shape == (min(w.C, 16), w.L)
    assert np.all(d[:, 0] == 0)
    assert np.all(np.diff(d, axis=1) > 0)          # sorted, distinct
    assert d.max() <= w.D
    if w.dirs == 2:                                 # DL and UL of a UE share delays
        assert np.array_equal(d[0::2], d[1::2])
    p = ttsynth.pdp(w, d)
    assert np.allclose(p.sum(axis=1), 1.0)
    assert np.all(np.diff(p, axis=1) < 0) or w.L == 1  # exponential decay with delay


def test_shard_independence():
    w = ttsynth.get("c3").scaled(n_per_call=256, calls=3)
    full_d = ttsynth.delays(w)
    full_g = ttsynth.snapshots(w, 0, w.C, 5)
    full_x = ttsynth.iq(w, 0, w.C, 2)
    for world in (2, 4, 8):
        for r in range(world):
            lo, hi = ttsynth.shard_ues(w, r, world)
            assert np.array_equal(ttsynth.delays(w, lo, hi), full_d[lo:hi])
            assert np.array_equal(ttsynth.snapshots(w, lo, hi, 5), full_g[lo:hi])
            assert np.array_equal(ttsynth.iq(w, lo, hi, 2), full_x[lo:hi])
    covered = sorted(c for r in range(8) for c in range(*ttsynth.shard_ues(w, r, 8)))
    assert covered == list(range(w.C))
    assert not np.array_equal(ttsynth.iq(w, 0, 2, 1), full_x[:2])  # other call, other draw


def test_input_statistics():
    w = ttsynth.get("c4").scaled(ues=4, n_per_call=1 << 16, calls=1)
    x = ttsynth.iq(w, 0, w.C, 0).astype(np.float64)
    assert abs((x ** 2).sum(-1).mean() - 1.0) < 0.01   # E|x|^2 = 1
    g = ttsynth.snapshots(w, 0, w.C, 2000).astype(np.float64)
    p = ttsynth.pdp(w, ttsynth.delays(w))
    ratio = (g ** 2).sum(-1).mean(axis=1) / p          # E|g_l|^2 = p_l
    assert np.all(np.abs(ratio - 1) < 0.15)
    assert abs(ratio.mean() - 1) < 0.02
