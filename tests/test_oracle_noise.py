"""Pins for the oracle's tt-normal-v1 transform (docs/tt-normal-v1.md §2-3):
exhaustive accuracy over every radius and every angle input against double libm,
and the moments / distribution of the resulting AWGN (SPEC S:257-259 style)."""
import math

import numpy as np
import pytest
from scipy import stats

import oracle


def _ulp32(x):
    return np.spacing(np.abs(x).astype(np.float32)).astype(np.float64)


def test_radius_exhaustive():
    rho = oracle.radius_all().astype(np.float64)  # A = 1 .. 2^24
    A = np.arange(1, (1 << 24) + 1, dtype=np.float64)
    exact = np.sqrt(-2.0 * np.log(A * 2.0 ** -24))
    err = np.abs(rho - exact)
    nz = exact > 0
    assert rho[-1] == 0.0 and exact[-1] == 0.0  # u = 1
    ulps = err[nz] / _ulp32(exact[nz])
    assert ulps.max() <= 2.0, ulps.max()
    # the largest radius: u = 2^-24 -> sqrt(48 ln 2)
    assert abs(rho[0] - math.sqrt(48 * math.log(2))) < 1e-6


def test_angle_exhaustive():
    cs = oracle.angle_all().astype(np.float64)
    j = np.arange(1 << 24, dtype=np.float64)
    theta = (np.pi / 2) * (j * 2.0 ** -22)
    ec = np.abs(cs[:, 0] - np.cos(theta))
    es = np.abs(cs[:, 1] - np.sin(theta))
    # absolute error within 2 ulp of 1 and the unit circle preserved
    assert ec.max() <= 2 * 2.0 ** -24 and es.max() <= 2 * 2.0 ** -24, (ec.max(), es.max())
    r = np.hypot(cs[:, 0], cs[:, 1])
    assert np.abs(r - 1).max() < 3e-7
    # exact quadrant values
    for q in range(4):
        c, s = cs[q << 22]
        assert (c, s) == [(1.0, 0.0), (0.0, 1.0), (-1.0, 0.0), (0.0, -1.0)][q] or \
            (abs(c) == abs([1, 0, -1, 0][q]) and abs(s) == abs([0, 1, 0, -1][q]))


@pytest.fixture(scope="module")
def noise_samples():
    sigma = 0.3
    w = np.concatenate([oracle.noise_block(12345, c, 0, 1 << 20, sigma) for c in range(10)]).astype(np.float64)
    return sigma, w


def test_noise_moments(noise_samples):
    sigma, w = noise_samples
    z = w[:, 0] + 1j * w[:, 1]
    n = len(z)
    assert abs(np.mean(np.abs(z) ** 2) / sigma ** 2 - 1) < 0.01          # E|w|^2 = sigma^2 +-1%
    assert abs(z.mean()) < 5 * sigma / math.sqrt(n)                        # mean 0
    assert abs(np.mean(z * z)) < 5 * sigma ** 2 / math.sqrt(n)             # circular: E[w^2] = 0
    for comp in (w[:, 0], w[:, 1]):
        k = stats.kurtosis(comp, fisher=False)
        assert abs(k - 3) < 0.05, k
    assert abs(np.corrcoef(w[:, 0], w[:, 1])[0, 1]) < 5 / math.sqrt(n)


def test_noise_ks(noise_samples):
    sigma, w = noise_samples
    sd = sigma / math.sqrt(2)
    for comp in (w[:2_000_000, 0], w[:2_000_000, 1]):
        p = stats.kstest(comp / sd, stats.norm.cdf).pvalue
        assert p > 1e-3, p


def test_noise_determinism_and_keys():
    a = oracle.noise_block(7, 3, 1000, 64, 1.0)
    b = oracle.noise_block(7, 3, 1000, 64, 1.0)
    assert np.array_equal(a, b)
    # any window of the stream reproduces the same samples (keyed by global sample)
    c = oracle.noise_block(7, 3, 990, 100, 1.0)
    assert np.array_equal(c[10:74], a)
    assert not np.array_equal(oracle.noise_block(7, 4, 1000, 64, 1.0), a)   # other channel
    assert not np.array_equal(oracle.noise_block(8, 3, 1000, 64, 1.0), a)   # other seed
    # sigma scales exactly by the float32 scale factor
    s = oracle.noise_scale(2.0)
    assert s == np.float32(2.0 * math.sqrt(0.5))
