"""Pins for the oracle's Philox4x32-10 (docs/tt-normal-v1.md §1) against things
other than itself: the Random123 known-answer vectors (tests/golden) and cuRAND's
host-side Philox4_32_10 generator (an independent library)."""
import ctypes as ct
import os

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "random123_philox4x32_10_kat.txt")


def _kat():
    rows = []
    for line in open(GOLDEN):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        w = [int(t, 16) for t in line.split()]
        rows.append((w[0:4], w[4:6], w[6:10]))
    return rows


@pytest.mark.parametrize("ctr,key,out", _kat())
def test_philox_known_answer(ctr, key, out):
    assert list(oracle.philox4x32_10(ctr, key)) == out


def _curand():
    for p in ("/usr/local/cuda/lib64/libcurand.so", "libcurand.so.10", "libcurand.so"):
        try:
            return ct.CDLL(p)
        except OSError:
            continue
    pytest.skip("libcurand not found")


@pytest.mark.parametrize("seed", [0, 1, 0x0123456789ABCDEF, 0xFFFFFFFF00000001])
def test_philox_vs_curand_host_generator(seed):
    """cuRAND's host Philox generator emits block b = Philox(ctr=(0,0,b,0), key=seed):
    this pins the key split (lo, hi) and the counter word that carries the channel id."""
    cr = _curand()
    gen = ct.c_void_p()
    CURAND_RNG_PSEUDO_PHILOX4_32_10 = 161
    assert cr.curandCreateGeneratorHost(ct.byref(gen), CURAND_RNG_PSEUDO_PHILOX4_32_10) == 0
    try:
        assert cr.curandSetPseudoRandomGeneratorSeed(gen, ct.c_ulonglong(seed)) == 0
        n = 4 * 64
        buf = (ct.c_uint32 * n)()
        assert cr.curandGenerate(gen, buf, ct.c_size_t(n)) == 0
        lib_words = np.frombuffer(buf, dtype=np.uint32).reshape(64, 4)
    finally:
        cr.curandDestroyGenerator(gen)
    key = [seed & 0xFFFFFFFF, seed >> 32]
    for b in range(64):
        assert list(oracle.philox4x32_10([0, 0, b, 0], key)) == list(lib_words[b]), b


def test_noise_counter_layout():
    """sample 2m takes words (r0, r1), sample 2m+1 takes (r2, r3) of counter (m lo, m hi, c, 0)."""
    seed, c, m = 0xABCDEF0123, 7, (1 << 33) + 5
    r = oracle.philox4x32_10([m & 0xFFFFFFFF, m >> 32, c, 0], [seed & 0xFFFFFFFF, seed >> 32])
    sc = oracle.noise_scale(1.0)
    w = oracle.noise_block(seed, c, 2 * m, 2, 1.0)
    z0 = oracle.normal_pair(int(r[0]), int(r[1]))
    z1 = oracle.normal_pair(int(r[2]), int(r[3]))
    assert w[0, 0] == np.float32(np.float32(z0[0]) * np.float32(sc))
    assert w[0, 1] == np.float32(np.float32(z0[1]) * np.float32(sc))
    assert w[1, 0] == np.float32(np.float32(z1[0]) * np.float32(sc))
    assert w[1, 1] == np.float32(np.float32(z1[1]) * np.float32(sc))
