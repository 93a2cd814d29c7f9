"""Pins of the oracle's sparse top-n convolution (NEXT f2, §III-C "convolution is
performed only with the top-n dominant taps at each time step"; R20), each
against something other than the oracle: SPEC's worked selection examples, a numpy
lexsort selection, the dense path at n >= L, Young's inequality bound, and a
pure-Python brute force of the interval-wise sum."""
import numpy as np
import pytest

import oracle


def test_spec_worked_example():
    """taps [0.1, 0.9, 0.05, 0.3], n = 2 -> bins {1, 3}."""
    g = np.array([[0.1, 0], [0.9, 0], [0.05, 0], [0.3, 0]], np.float32)
    assert list(np.flatnonzero(oracle.select_top_n([0, 1, 2, 3], g, 2))) == [1, 3]


def test_spec_tie_goes_to_smaller_bin():
    """equal-magnitude taps at bins 2 and 5, n = 1 -> bin 2 (here with the
    taps listed out of delay order and with equal |g| from different phases)."""
    d = np.array([5, 9, 2], np.int32)
    g = np.array([[0.6, 0.8], [0.1, 0.0], [-1.0, 0.0]], np.float32)  # |g| = 1, 0.1, 1
    assert list(np.flatnonzero(oracle.select_top_n(d, g, 1))) == [2]


@pytest.mark.parametrize("L,n", [(8, 3), (23, 10), (48, 20), (64, 64), (5, 9)])
def test_selection_matches_lexsort(L, n):
    rng = np.random.default_rng(L * 100 + n)
    for _ in range(20):
        d = np.sort(rng.choice(4 * L + 1, L, replace=False)).astype(np.int32)
        g = rng.standard_normal((L, 2)).astype(np.float32)
        g[rng.integers(0, L, 3)] = g[0]  # some exact ties
        m = (g[:, 0] * g[:, 0]).astype(np.float32) + (g[:, 1] * g[:, 1]).astype(np.float32)
        order = np.lexsort((np.arange(L), d, -m.astype(np.float64)))
        ref = np.zeros(L, bool)
        ref[order[:min(n, L)]] = True
        assert np.array_equal(oracle.select_top_n(d, g, n), ref)


def _case(rng, C=2, L=12, D=60, S=32, N=400):
    K = (N - 1) // S + 2
    d = np.stack([np.sort(rng.choice(D + 1, L, replace=False)) for _ in range(C)]).astype(np.int32)
    g = rng.standard_normal((C, K, L, 2)).astype(np.float32)
    x = rng.standard_normal((C, N, 2)).astype(np.float32)
    return d, S, g, x, N


def test_n_at_least_L_is_the_dense_path():
    d, S, g, x, N = _case(np.random.default_rng(0))
    dense = oracle.convolve(d, S, g, 0, x, 0, 0, N)
    for n in (d.shape[1], d.shape[1] + 5):
        assert np.array_equal(oracle.convolve(d, S, g, 0, x, 0, 0, N, top_n=n), dense)


def test_brute_force_interval_sum():
    """Pure-Python double loop: each output sums the taps numpy selects for its interval."""
    rng = np.random.default_rng(3)
    d, S, g, x, N = _case(rng, C=1, L=6, D=20, S=8, N=70)
    n_top = 2
    got = oracle.convolve(d, S, g, 0, x, 0, 0, N, top_n=n_top)[0]
    xc = x[0, :, 0].astype(np.float64) + 1j * x[0, :, 1]
    gc = g[0, ..., 0].astype(np.float64) + 1j * g[0, ..., 1]
    for n in range(N):
        k, j = divmod(n, S)
        m = (g[0, k, :, 0] * g[0, k, :, 0]).astype(np.float32) + (g[0, k, :, 1] * g[0, k, :, 1]).astype(np.float32)
        keep = np.lexsort((np.arange(6), d[0], -m.astype(np.float64)))[:n_top]
        acc = 0j
        for l in keep:
            h = gc[k, l] + (j / S) * (gc[k + 1, l] - gc[k, l])
            if n - d[0, l] >= 0:
                acc += h * xc[n - d[0, l]]
        assert abs(got[n] - acc) <= 1e-12 * max(1.0, abs(acc))


def test_young_bound():
    """with time-invariant taps, ||y_full - y_sparse||_2 <= ||x||_2 * sum of the
    omitted |h_l| (Young's inequality for the convolution with the omitted taps)."""
    rng = np.random.default_rng(7)
    d, S, g, x, N = _case(rng, C=1, L=16, D=80, S=64, N=600)
    g[:] = g[:, :1]  # every snapshot equal -> h constant
    n_top = 13
    full = oracle.convolve(d, S, g, 0, x, 0, 0, N)[0]
    sparse = oracle.convolve(d, S, g, 0, x, 0, 0, N, top_n=n_top)[0]
    sel = oracle.select_top_n(d[0], g[0, 0], n_top)
    omitted = np.abs(g[0, 0, ~sel, 0].astype(np.float64) + 1j * g[0, 0, ~sel, 1]).sum()
    xn = np.linalg.norm(x[0, :, 0].astype(np.float64) + 1j * x[0, :, 1])
    err = np.linalg.norm(full - sparse)
    assert 0 < err <= xn * omitted
