"""Pins for the oracle's convolution (oracle/tt_oracle.c; NS formula, P:305-306,
P:309) against what the paper and mathematics fix, not against itself:
closed forms, special cases that reduce to library routines (numpy.convolve,
numpy.interp + a dense matrix product), invariants (linearity, window
independence) and a closed-form second moment."""
import math

import numpy as np
import pytest

import oracle
import ttsynth


def _cplx(a):
    return a[..., 0].astype(np.float64) + 1j * a[..., 1].astype(np.float64)


def _rand(rng, *shape):
    return rng.standard_normal((*shape, 2)).astype(np.float32)


def test_identity_single_unit_tap():
    """L=1, d=0, g == 1 -> y == x (OAI's 1-tap special case)."""
    rng = np.random.default_rng(0)
    N, S = 1000, 64
    x = _rand(rng, 2, N)
    g = np.zeros((2, N // S + 2, 1, 2), np.float32)
    g[..., 0] = 1.0
    y = oracle.convolve([[0], [0]], S, g, 0, x, 0, 0, N)
    assert np.array_equal(y, _cplx(x))


def test_pure_delay_zero_history():
    """L=1, d=D, g == 1 -> y[n] = x[n-D], zeros for n < D."""
    rng = np.random.default_rng(1)
    N, S, D = 500, 32, 37
    x = _rand(rng, 1, N)
    g = np.zeros((1, N // S + 2, 1, 2), np.float32)
    g[..., 0] = 1.0
    y = oracle.convolve([[D]], S, g, 0, x, 0, 0, N)[0]
    assert np.all(y[:D] == 0)
    assert np.array_equal(y[D:], _cplx(x)[0, : N - D])
    # SPEC example: taps [0, 1], input [a, b, c] -> [0, a, b]
    x3 = np.array([[[1, 2], [3, 4], [5, 6]]], np.float32)
    g2 = np.zeros((1, 2, 2, 2), np.float32)
    g2[..., 1, 0] = 1.0
    y3 = oracle.convolve([[0, 1]], 4, g2, 0, x3, 0, 0, 3)[0]
    assert np.array_equal(y3, np.array([0, 1 + 2j, 3 + 4j]))


def test_scalar_fading_is_piecewise_linear_through_snapshots():
    """x == 1, one tap at d=0: y is the tap gain itself. It must pass through the
    snapshots exactly at n = kS, be linear inside each interval (constant first
    difference (g_{k+1} - g_k)/S), and be continuous across interval boundaries."""
    rng = np.random.default_rng(2)
    S, K = 16, 9
    N = S * (K - 1)
    g = _rand(rng, 1, K, 1)
    x = np.zeros((1, N, 2), np.float32)
    x[..., 0] = 1.0
    y = oracle.convolve([[0]], S, g, 0, x, 0, 0, N)[0]
    gk = _cplx(g)[0, :, 0]
    for k in range(K - 1):
        assert y[k * S] == gk[k]
        seg = y[k * S:(k + 1) * S]
        d1 = np.diff(np.concatenate([seg, [gk[k + 1]]]))
        assert np.allclose(d1, (gk[k + 1] - gk[k]) / S, rtol=0, atol=1e-12)


def test_time_index_is_output_time():
    """Unit impulse at m, one tap at delay d with time-varying gains: the only
    non-zero output is y[m + d], and it equals the tap gain at time m + d (the
    scalar-fading output there), not at time m (reading R1)."""
    rng = np.random.default_rng(3)
    S, K, d, m = 8, 12, 5, 13
    N = S * (K - 1)
    g = _rand(rng, 1, K, 1)
    x = np.zeros((1, N, 2), np.float32)
    x[0, m, 0] = 1.0
    y = oracle.convolve([[d]], S, g, 0, x, 0, 0, N)[0]
    nz = np.flatnonzero(y)
    assert list(nz) == [m + d]
    ones = np.zeros((1, N, 2), np.float32)
    ones[..., 0] = 1.0
    gain = oracle.convolve([[0]], S, g, 0, ones, 0, 0, N)[0]
    assert y[m + d] == gain[m + d]
    assert y[m + d] != gain[m]


@pytest.mark.parametrize("L,D", [(1, 0), (4, 12), (20, 64)])
def test_time_invariant_equals_numpy_convolve(L, D):
    """All snapshots equal -> y = numpy.convolve(x, h_dense)[:N]."""
    rng = np.random.default_rng(4 + L)
    N, S = 1024, 64
    K = N // S + 2
    d = np.concatenate([[0], np.sort(rng.choice(np.arange(1, D + 1), L - 1, replace=False))]) if L > 1 else [0]
    g0 = _rand(rng, 1, 1, L)
    g = np.repeat(g0, K, axis=1)
    x = _rand(rng, 1, N)
    y = oracle.convolve([d], S, g, 0, x, 0, 0, N)[0]
    h_dense = np.zeros(max(d) + 1, np.complex128)
    for l in range(L):
        h_dense[d[l]] += _cplx(g0)[0, 0, l]
    ref = np.convolve(_cplx(x)[0], h_dense)[:N]
    assert np.max(np.abs(y - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))


def test_brute_force_matrix_with_library_interpolation():
    """Tiny inputs: build the time-varying convolution matrix H (H[n, n-d_l] += h_l[n])
    with h_l[n] from numpy.interp over the snapshot instants kS, then y = H x."""
    rng = np.random.default_rng(5)
    for trial in range(20):
        C, L, S = 2, int(rng.integers(1, 9)), int(rng.integers(1, 9))
        N = int(rng.integers(1, 65))
        K = (N - 1) // S + 2
        d = np.stack([np.sort(rng.choice(20, L, replace=False)) for _ in range(C)])
        g = _rand(rng, C, K, L)
        x = _rand(rng, C, N)
        y = oracle.convolve(d, S, g, 0, x, 0, 0, N)
        for c in range(C):
            H = np.zeros((N, N), np.complex128)
            tk = np.arange(K) * S
            for l in range(L):
                gc = _cplx(g)[c, :, l]
                h = np.interp(np.arange(N), tk, gc.real) + 1j * np.interp(np.arange(N), tk, gc.imag)
                for n in range(N):
                    if n - d[c, l] >= 0:
                        H[n, n - d[c, l]] += h[n]
            ref = H @ _cplx(x)[c]
            assert np.allclose(y[c], ref, rtol=0, atol=1e-12), (trial, c)


def test_linearity():
    """y(a x1 + b x2) = a y(x1) + b y(x2) for sigma = 0."""
    rng = np.random.default_rng(6)
    N, S, L = 700, 50, 6
    d = [[0, 2, 5, 9, 14, 30]]
    g = _rand(rng, 1, N // S + 2, L)
    # inputs on a 2^-10 grid so that a x1 + b x2 is exact in float32
    x1 = np.round(_rand(rng, 1, N).astype(np.float64) * 1024) / 1024
    x2 = np.round(_rand(rng, 1, N).astype(np.float64) * 1024) / 1024
    a, b = 0.5, -2.0
    x3 = (a * x1 + b * x2).astype(np.float32)
    assert np.array_equal(x3.astype(np.float64), a * x1 + b * x2)
    y1 = oracle.convolve(d, S, g, 0, x1.astype(np.float32), 0, 0, N)
    y2 = oracle.convolve(d, S, g, 0, x2.astype(np.float32), 0, 0, N)
    y3 = oracle.convolve(d, S, g, 0, x3, 0, 0, N)
    assert np.allclose(y3, a * y1 + b * y2, rtol=0, atol=1e-12)


def test_window_independence_and_points():
    """Outputs depend only on the stream, not on which window of it is stored or on
    how outputs are requested (the streaming property S:263 for a stateless oracle);
    a missing needed sample or snapshot is an error, not a silent zero."""
    rng = np.random.default_rng(7)
    C, L, S, N = 3, 5, 32, 400
    d = np.stack([np.sort(rng.choice(40, L, replace=False)) for _ in range(C)])
    g = _rand(rng, C, N // S + 2, L)
    x = _rand(rng, C, N)
    full = oracle.convolve(d, S, g, 0, x, 0, 0, N, sigma=0.1, seed=9)
    part = oracle.convolve(d, S, g, 0, x[:, 200:], 200, 250, 150, sigma=0.1, seed=9)
    assert np.array_equal(part, full[:, 250:])
    # snapshot window k0 > 0
    k0 = 250 // S
    part2 = oracle.convolve(d, S, g[:, k0:], k0, x, 0, 250, 150, sigma=0.1, seed=9)
    assert np.array_equal(part2, full[:, 250:])
    cs = rng.integers(0, C, 50)
    ns = rng.integers(0, N, 50)
    pts = oracle.convolve_points(d, S, g, 0, x, 0, cs, ns, sigma=0.1, seed=9)
    assert np.array_equal(pts, full[cs, ns])
    with pytest.raises(oracle.OracleError):
        oracle.convolve(d, S, g, 0, x[:, 200:], 200, 210, 10)  # needs x[210 - 39] < 200
    with pytest.raises(oracle.OracleError):
        oracle.convolve(d, S, g[:, :3], 0, x, 0, 0, N)


def test_noise_only_output_is_the_noise():
    """x == 0 -> y == w exactly (docs/tt-normal-v1.md §3)."""
    N, S = 300, 16
    g = np.ones((2, N // S + 2, 3, 2), np.float32)
    x = np.zeros((2, N, 2), np.float32)
    y = oracle.convolve([[0, 1, 2], [0, 3, 4]], S, g, 0, x, 0, 0, N, sigma=0.7, seed=42, c_offset=10)
    for c in range(2):
        w = oracle.noise_block(42, 10 + c, 0, N, 0.7)
        assert np.array_equal(y[c], _cplx(w))


def test_received_power_closed_form():
    """iid CN(0,1) input, iid Rayleigh snapshots CN(0, p_l) at distinct delays, linear
    interpolation: E|y|^2 = (2/3 + 1/(3 S^2)) sum_l p_l + sigma^2 (derivation:
    E[(1-a)^2 + a^2] over a = j/S, j = 0..S-1), and the per-tap mean power follows
    the power-delay profile (north_star PDP pin)."""
    w = ttsynth.get("c3").scaled(ues=32, dirs=1, n_per_call=8192, calls=1, S=4)
    C = w.C
    d = ttsynth.delays(w)
    g = ttsynth.snapshots(w, 0, C, w.K_total)
    x = ttsynth.iq(w, 0, C, 0)
    sigma = 0.5
    y = oracle.convolve(d, w.S, g, 0, x, 0, 0, w.n_per_call, sigma=sigma, seed=3)
    yy = y[:, 1024:]  # skip the zero-history ramp (max delay 600)
    factor = 2.0 / 3.0 + 1.0 / (3.0 * w.S ** 2)
    # finite-sample reference: snapshot powers actually drawn (removes snapshot variance)
    p_emp = (np.abs(_cplx(g)) ** 2).mean(axis=1)                      # [C][L]
    expect = factor * p_emp.sum(axis=1).mean() + sigma ** 2
    got = (np.abs(yy) ** 2).mean()
    assert abs(got / expect - 1) < 0.03, (got, expect)
    # PDP: per-tap empirical mean |g|^2 / p_l -> 1
    p = ttsynth.pdp(w, d)
    ratio = (p_emp / p).mean(axis=0)
    assert np.all(np.abs(ratio - 1) < 5 * math.sqrt(1.0 / (C * w.K_total)) * 1.5)
    # single tap, x == 1: time-average |h|^2 = factor * p_l exactly in expectation
    ones = np.zeros((C, w.n_per_call, 2), np.float32)
    ones[..., 0] = 1.0
    h = oracle.convolve(np.zeros((C, 1), np.int32), w.S, g[:, :, :1], 0, ones, 0, 0, w.n_per_call)
    emp = (np.abs(h) ** 2).mean() / p[:, 0].mean()
    assert abs(emp / factor - 1) < 0.03, emp
