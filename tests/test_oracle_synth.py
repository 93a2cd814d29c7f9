"""Pins of the oracle's channel-state synthesis (NEXT f3: Jakes sum-of-sinusoids per
path + two-bin fractional-delay split; §IV; R21), each against
something other than the oracle: zero Doppler freezes the fading, unit mean power,
the Clarke/Jakes autocorrelation J0(2 pi nu tau) from scipy's Bessel function, SPEC's
resampling examples and first-moment preservation, determinism."""
import numpy as np
import pytest
from scipy.special import j0

import oracle


def _c(g):
    return g[..., 0].astype(np.float64) + 1j * g[..., 1]


def test_zero_doppler_is_constant():
    """f_d = 0 -> constant gain sequence."""
    d, g = oracle.synth_jakes([[0.0, 2.5, 7.0]], [[0.5, 0.3, 0.2]], 32, 0.0, 9, 0, 20)
    assert np.array_equal(g, np.broadcast_to(g[:, :1], g.shape))


def test_unit_mean_power():
    """unit mean power; sample mean within 3 %."""
    C, P = 40, 50
    tau = np.arange(P, dtype=np.float32)[None].repeat(C, 0) * 3
    d, g = oracle.synth_jakes(tau, np.ones((C, P), np.float32), 32, 0.02, 5, 0, 400)
    p = np.abs(_c(g[:, :, 0::2])) ** 2  # on-grid paths: all power in the first bin
    assert abs(p.mean() - 1.0) < 0.03
    assert np.all(g[:, :, 1::2] == 0)


@pytest.mark.parametrize("nu", [0.0162, 0.1944])
def test_autocorrelation_is_bessel_j0(nu):
    """normalised autocorrelation at lags {1, 2, 5, 10} steps within 0.05
    of J0(2 pi f_d tau) (f_d = 16.2 / 194.4 Hz at a 1 ms step, i.e. nu in cycles/step)."""
    C, P, K = 20, 50, 1500
    tau = np.zeros((C, P), np.float32)
    d, g = oracle.synth_jakes(tau, np.ones((C, P), np.float32), 32, nu, 77, 0, K)
    a = _c(g[:, :, 0::2])  # [C][K][P]
    p0 = np.mean(np.abs(a) ** 2)
    for lag in (1, 2, 5, 10):
        r = np.mean(a[:, lag:] * np.conj(a[:, :-lag])) / p0
        assert abs(r.real - j0(2 * np.pi * nu * lag)) < 0.05, (lag, r, j0(2 * np.pi * nu * lag))


def test_resampling_examples_and_first_moment():
    """on-grid path -> one bin; path at 1.5 bins -> two equal halves; the
    complex-gain-weighted first delay moment is preserved."""
    tau = np.array([[3.0, 1.5, 12.3125]], np.float32)
    d, g = oracle.synth_jakes(tau, np.array([[0.2, 0.3, 0.5]], np.float32), 16, 0.0, 3, 0, 2)
    assert list(d[0]) == [3, 4, 1, 2, 12, 13]
    gc = _c(g[0, 0])
    assert gc[1] == 0                       # on grid
    assert gc[2] == gc[3]                   # midpoint split
    for p in range(3):
        tot = gc[2 * p] + gc[2 * p + 1]
        moment = d[0, 2 * p] * gc[2 * p] + d[0, 2 * p + 1] * gc[2 * p + 1]
        assert abs(moment - tau[0, p] * tot) <= 1e-6 * abs(tot) * (tau[0, p] + 1)


def test_determinism_and_keys():
    args = ([[0.0, 4.5]], [[0.6, 0.4]], 24, 0.05)
    a = oracle.synth_jakes(*args, 11, 0, 30)[1]
    assert np.array_equal(a, oracle.synth_jakes(*args, 11, 0, 30)[1])
    assert not np.array_equal(a, oracle.synth_jakes(*args, 12, 0, 30)[1])
    assert not np.array_equal(a, oracle.synth_jakes(*args, 11, 0, 30, c_offset=1)[1])
    # snapshot k depends only on k: a later window equals the slice of a long run
    assert np.array_equal(a[:, 10:20], oracle.synth_jakes(*args, 11, 10, 10)[1])
