"""Pins of the oracle's group sums (NEXT f1 UL aggregation, f4 multi-gNB links), each
against something other than the oracle itself: SPEC's worked aggregation example,
the closed form of pure-delay links, and the vanilla (serial per-UE) == optimised
(grouped) equivalence."""
import numpy as np
import pytest

import oracle


def _unit_taps(gains_per_channel, K):
    """gains [C][K][1][2] holding a constant real gain per channel."""
    g = np.zeros((len(gains_per_channel), K, 1, 2), np.float32)
    for c, v in enumerate(gains_per_channel):
        g[c, :, 0, 0] = v
    return g


def test_spec_two_ues_taps_1_and_2_give_three_times_the_frame():
    """2 UEs with taps [1] and [2] on identical unit uplink frames -> aggregate =
    3x frame ("only then aggregates them")."""
    N, S = 257, 16
    K = (N - 1) // S + 2
    frame = np.zeros((2, N, 2), np.float32)
    frame[..., 0] = 1.0
    y = oracle.convolve(np.zeros((2, 1), np.int32), S, _unit_taps([1.0, 2.0], K), 0, frame, 0, 0, N)
    agg = oracle.aggregate(y, 2)
    assert agg.shape == (1, N)
    assert np.array_equal(agg[0], np.full(N, 3.0 + 0j))


def test_links_with_pure_delays_sum_to_delayed_sources():
    """f4 closed form: UE u receives B gNB streams through single unit taps at delays
    d_b -> y_u[n] = sum_b x_b[n - d_b] (zero before the stream starts)."""
    rng = np.random.default_rng(1)
    B, N, S = 3, 300, 32
    K = (N - 1) // S + 2
    xg = rng.standard_normal((B, N, 2)).astype(np.float32)
    d = np.array([[0], [5], [17]], np.int32)
    y = oracle.convolve(d, S, _unit_taps([1.0] * B, K), 0, xg, 0, 0, N)
    agg = oracle.aggregate(y, B)[0]
    ref = np.zeros(N, np.complex128)
    for b in range(B):
        xb = xg[b, :, 0].astype(np.float64) + 1j * xg[b, :, 1]
        ref[d[b, 0]:] += xb[:N - d[b, 0]]
    assert np.allclose(agg, ref, rtol=0, atol=1e-12)


@pytest.mark.parametrize("C,G", [(6, 3), (6, 1), (8, 8)])
def test_vanilla_serial_equals_grouped(C, G):
    """S:320 mode equivalence: convolving each UE on its own and summing serially at
    the 'gNB' equals the grouped sum of one multi-channel run; groups are consecutive
    channels."""
    rng = np.random.default_rng(C * 10 + G)
    L, D, S, N = 5, 40, 64, 500
    K = (N - 1) // S + 2
    d = np.stack([np.sort(rng.choice(D + 1, L, replace=False)) for _ in range(C)]).astype(np.int32)
    g = rng.standard_normal((C, K, L, 2)).astype(np.float32)
    x = rng.standard_normal((C, N, 2)).astype(np.float32)
    grouped = oracle.aggregate(oracle.convolve(d, S, g, 0, x, 0, 0, N), G)
    for gi in range(C // G):
        serial = np.zeros(N, np.complex128)
        for c in range(gi * G, (gi + 1) * G):
            serial += oracle.convolve(d[c:c + 1], S, g[c:c + 1], 0, x[c:c + 1], 0, 0, N)[0]
        assert np.allclose(grouped[gi], serial, rtol=1e-13, atol=1e-13)


def test_aggregate_rejects_bad_group():
    with pytest.raises(oracle.OracleError):
        oracle.aggregate(np.zeros((5, 3)), 2)
