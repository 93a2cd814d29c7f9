"""NEXT rows f1 (UL aggregation at the gNB) and f4 (multi-gNB links) on the GPU,
through the C ABI: tt_channel_apply_aggregate and tt_channel_set_input_map.

Parity: the group sums match the oracle (double sums of double channel outputs)
within north_star's tolerances; the fused chunk sums equal, bit for bit, a float32
left-to-right emulation of the documented order over the same call's per-channel
outputs; results are bit-identical for any call split and on every kernel path."""
import numpy as np
import pytest

import oracle
import ttsynth
from harness import Run, compare, to_c

pytestmark = pytest.mark.gpu

CHUNK = 8  # TT_AGG_CHUNK


def _chunked_sum_f32(y, G):
    """The documented order: chunks of CHUNK channels summed left to right in float32,
    then the chunk sums left to right."""
    C, N, _ = y.shape
    out = np.empty((C // G, N, 2), np.float32)
    for g in range(C // G):
        s = None
        for q0 in range(0, G, CHUNK):
            p = y[g * G + q0].copy()
            for k in range(1, min(CHUNK, G - q0)):
                p = (p + y[g * G + q0 + k]).astype(np.float32)
            s = p if s is None else (s + p).astype(np.float32)
        out[g] = s
    return out


def _run_aggregate(run, device, G, calls, rows=None, x_rows=None, with_out=True, device_clock=False):
    import torch

    from paper_2601_08217_b200 import Channel

    ch = Channel(run.delays, run.w.S, seed=run.seed, snapshot_capacity=run.K, channel_offset=run.c_lo, device=device)
    try:
        ch.load_snapshots(torch.from_numpy(run.gains).to(device), 0)
        if device_clock:
            ch.set_device_clock(True)
        src = run.x if x_rows is None else x_rows
        if rows is not None:
            ch.set_input_map(rows, src.shape[0])
        ys, aggs, pos = [], [], 0
        for n in calls:
            xs = torch.from_numpy(np.ascontiguousarray(src[:, pos:pos + n])).to(device)
            out = torch.empty((run.C, n, 2), dtype=torch.float32, device=device) if with_out else None
            agg = ch.apply_aggregate(xs, G, out=out, noise_sigma=run.sigma)
            aggs.append(agg.cpu().numpy())
            if with_out:
                ys.append(out.cpu().numpy())
            pos += n
        torch.cuda.synchronize()
    finally:
        ch.close()
    return (np.concatenate(ys, axis=1) if with_out else None), np.concatenate(aggs, axis=1)


@pytest.mark.parametrize("G", [1, 2, 16, 17, 40])
@pytest.mark.parametrize("snr", [None, 15.0])
def test_ul_aggregation_parity_and_order(cuda_device, G, snr):
    """f1: agg[g] = sum of the group's channel outputs: oracle parity, and the fused
    chunk sums equal the float32 emulation of the documented order bit for bit."""
    C = G * (4 if G < 16 else 2)  # groups of G consecutive channels
    w = ttsynth.get("c3").scaled(ues=C, dirs=1, n_per_call=7_001, calls=1, snr_db=snr)
    run = Run(w, seed=31)
    y, agg = _run_aggregate(run, cuda_device, G, [7_001])
    assert np.array_equal(agg, _chunked_sum_f32(y, G))
    ref = oracle.aggregate(run.oracle(), G)
    compare(agg, ref, f"aggregate G={G}")


def test_aggregation_streaming_and_kernel_paths_bit_identical(cuda_device, monkeypatch):
    w = ttsynth.get("c4").scaled(ues=12, dirs=2, n_per_call=9_000, calls=1)
    run = Run(w, seed=5)
    _, one = _run_aggregate(run, cuda_device, 24, [9_000], with_out=False)
    _, split = _run_aggregate(run, cuda_device, 24, [1, 4_095, 17, 4_887], with_out=False)
    assert np.array_equal(one, split)
    monkeypatch.setenv("TT_KERNEL", "generic")
    _, gen = _run_aggregate(run, cuda_device, 24, [9_000], with_out=False)
    monkeypatch.delenv("TT_KERNEL")
    assert np.array_equal(one, gen)
    compare(one, oracle.aggregate(run.oracle(), 24), "c4 UL aggregate")


def test_aggregation_and_links_in_device_clock_mode(cuda_device):
    """Device-clock mode (the graph-capturable stream position) gives the same per-channel
    outputs and group sums as host-clock calls, for the f1 aggregate and the f4 links."""
    w = ttsynth.get("c4").scaled(ues=12, dirs=2, n_per_call=4_096, calls=3)
    run = Run(w, seed=15)
    calls = [4_096] * 3
    y0, a0 = _run_aggregate(run, cuda_device, 24, calls)
    y1, a1 = _run_aggregate(run, cuda_device, 24, calls, device_clock=True)
    assert np.array_equal(y0, y1) and np.array_equal(a0, a1)
    U, B = 4, 3
    wl = ttsynth.get("c3").scaled(ues=U * B, dirs=1, n_per_call=2_048, calls=2)
    rl = Run(wl, seed=16)
    xg = ttsynth.iq(wl, 0, B, 0, 4_096)
    rows = np.tile(np.arange(B, dtype=np.int32), U)
    rl.x = xg[rows]
    y0, a0 = _run_aggregate(rl, cuda_device, B, [2_048, 2_048], rows=rows, x_rows=xg)
    y1, a1 = _run_aggregate(rl, cuda_device, B, [2_048, 2_048], rows=rows, x_rows=xg, device_clock=True)
    assert np.array_equal(y0, y1) and np.array_equal(a0, a1)
    compare(y0, rl.oracle(), "links")


def test_multi_gnb_links(cuda_device):
    """f4: U UEs x B gNBs links (c = u B + b) reading the B gNB streams
    through the input map; agg[u] = the UE's received sum over its links."""
    U, B = 5, 3
    w = ttsynth.get("c3").scaled(ues=U * B, dirs=1, n_per_call=6_000, calls=1, snr_db=20.0)
    run = Run(w, seed=77)
    xg = ttsynth.iq(w, 0, B, 0)  # the B gNB transmit streams
    rows = np.tile(np.arange(B, dtype=np.int32), U)
    run.x = xg[rows]  # what each link sees, for the oracle
    y, agg = _run_aggregate(run, cuda_device, B, [2_500, 3_500], rows=rows, x_rows=xg)
    compare(y, run.oracle(), "links")
    compare(agg, oracle.aggregate(run.oracle(), B), "UE sums")
    assert np.array_equal(agg, _chunked_sum_f32(y, B))


def test_input_map_plain_apply_and_errors(cuda_device):
    import torch

    from paper_2601_08217_b200 import Channel, TTError

    w = ttsynth.get("c3").scaled(ues=4, dirs=1, n_per_call=3_000, calls=1)
    run = Run(w, seed=3)
    xg = run.x[:2].copy()
    rows = np.array([1, 0, 1, 1], np.int32)
    ch = Channel(run.delays, w.S, seed=3, snapshot_capacity=run.K, device=cuda_device)
    ch.load_snapshots(torch.from_numpy(run.gains).to(cuda_device), 0)
    with pytest.raises(TTError, match="INVALID_ARG"):
        ch.set_input_map(np.array([0, 1, 2, 5], np.int32), 3)
    ch.set_input_map(rows, 2)
    y = ch.apply(torch.from_numpy(xg).to(cuda_device), noise_sigma=run.sigma).cpu().numpy()
    xh = torch.zeros((4, 10, 2)).pin_memory()
    with pytest.raises(TTError, match="UNSUPPORTED"):
        ch.apply_host(xh, torch.zeros_like(xh).pin_memory())
    with pytest.raises(ValueError):
        ch.apply_aggregate(torch.from_numpy(xg).to(cuda_device), 3)
    ch.close()
    run.x = xg[rows]
    compare(y, run.oracle(), "mapped apply")


def _run_sparse(run, device, top_n, calls, set_before_load=True):
    import torch

    from paper_2601_08217_b200 import Channel

    ch = Channel(run.delays, run.w.S, seed=run.seed, snapshot_capacity=run.K, channel_offset=run.c_lo, device=device)
    try:
        if set_before_load:
            ch.set_top_n(top_n)
        ch.load_snapshots(torch.from_numpy(run.gains).to(device), 0)
        if not set_before_load:
            ch.set_top_n(top_n)
        assert ch.info().top_n == (top_n if 0 < top_n < run.w.L else 0)
        out, pos = [], 0
        for n in calls:
            xs = torch.from_numpy(np.ascontiguousarray(run.x[:, pos:pos + n])).to(device)
            out.append(ch.apply(xs, noise_sigma=run.sigma).cpu().numpy())
            pos += n
        torch.cuda.synchronize()
    finally:
        ch.close()
    return np.concatenate(out, axis=1)


@pytest.mark.parametrize("name,kw,top_n", [
    ("c4", dict(ues=2, n_per_call=12_000, calls=1), 20),        # one interval per warp (S=256, R=8)
    ("c4", dict(ues=2, n_per_call=12_000, calls=1), 1),
    ("c5-L64", dict(ues=2, n_per_call=9_000), 16),               # S=128: two intervals per warp
    ("c3", dict(ues=2, n_per_call=8_000, calls=1), 10),
    ("c2", dict(ues=2, n_per_call=5_000), 22),
])
def test_sparse_top_n_parity(cuda_device, name, kw, top_n):
    """f2: each interval sums its top-n taps; oracle parity (same float32
    selection rule), any call split bit-identical, tiled == generic bit for bit."""
    w = ttsynth.get(name).scaled(**kw)
    run = Run(w, seed=13)
    N = run.N
    y = _run_sparse(run, cuda_device, top_n, [N])
    ref = oracle.convolve(run.delays, w.S, run.gains, 0, run.x, 0, 0, N, sigma=run.sigma, seed=run.seed,
                          top_n=top_n)
    compare(y, ref, f"{name} top-{top_n}")
    assert np.array_equal(_run_sparse(run, cuda_device, top_n, [N // 3, 7, N - N // 3 - 7]), y)
    assert np.array_equal(_run_sparse(run, cuda_device, top_n, [N], set_before_load=False), y)


def test_sparse_n_equal_L_is_dense_and_generic_path(cuda_device, monkeypatch):
    w = ttsynth.get("c4").scaled(ues=2, n_per_call=9_000, calls=1)
    run = Run(w, seed=2)
    dense = run.gpu(cuda_device)
    assert np.array_equal(_run_sparse(run, cuda_device, w.L, [run.N]), dense)
    assert np.array_equal(_run_sparse(run, cuda_device, 0, [run.N]), dense)
    sp = _run_sparse(run, cuda_device, 17, [run.N])
    monkeypatch.setenv("TT_KERNEL", "generic")
    assert np.array_equal(_run_sparse(run, cuda_device, 17, [run.N]), sp)
    monkeypatch.delenv("TT_KERNEL")


@pytest.mark.parametrize("nu,M", [(0.0, 16), (4e-4, 32), (0.05, 32)])
def test_jakes_synthesis_parity(cuda_device, nu, M):
    """f3: GPU-synthesised snapshots vs the oracle's double-precision Jakes
    (same Philox draws) — relative RMS <= 1e-5 per channel; grid delays identical;
    windows of a long run (large k) keep the accuracy."""
    import torch

    from paper_2601_08217_b200 import synth_jakes

    rng = np.random.default_rng(4)
    C, P = 6, 12
    tau = np.sort(rng.uniform(0, 300, (C, P)), axis=1).astype(np.float32)
    tau[:, 0] = 0.0
    pw = rng.uniform(0.1, 1.0, (C, P)).astype(np.float32)
    pw /= pw.sum(axis=1, keepdims=True)
    for k0, K in ((0, 300), (1_000_000, 50)):
        d, g = synth_jakes(tau, pw, M, nu, seed=99, first_index=k0, count=K, channel_offset=3, device=cuda_device)
        dr, gr = oracle.synth_jakes(tau, pw, M, nu, 99, k0, K, c_offset=3)
        assert np.array_equal(d, dr)
        gg = to_c(g.cpu().numpy())
        gref = to_c(gr)
        for c in range(C):
            err = np.linalg.norm(gg[c] - gref[c]) / np.linalg.norm(gref[c])
            assert err <= 1e-5, (c, k0, err)


def test_jakes_slot_by_slot_calls(cuda_device):
    """Slot-by-slot synthesis: split windows equal one call bit for bit, and a changed
    path delay, power or seed between calls is picked up (no stale per-device state)."""
    from paper_2601_08217_b200 import synth_jakes

    rng = np.random.default_rng(5)
    C, P, M, nu = 5, 8, 16, 0.003
    tau = np.sort(rng.uniform(0, 200, (C, P)), axis=1).astype(np.float32)
    pw = rng.uniform(0.1, 1.0, (C, P)).astype(np.float32)
    _, whole = synth_jakes(tau, pw, M, nu, seed=9, first_index=0, count=96, device=cuda_device)
    parts = [synth_jakes(tau, pw, M, nu, seed=9, first_index=k, count=32, device=cuda_device)[1]
             for k in (0, 32, 64)]
    import torch

    assert np.array_equal(torch.cat(parts, dim=1).cpu().numpy(), whole.cpu().numpy())
    for t2, p2, s2 in ((tau + np.float32(0.5), pw, 9), (tau, pw * np.float32(2), 9), (tau, pw, 10)):
        _, g = synth_jakes(t2, p2, M, nu, seed=s2, first_index=0, count=32, device=cuda_device)
        _, gr = oracle.synth_jakes(t2, p2, M, nu, s2, 0, 32)
        gg, gref = to_c(g.cpu().numpy()), to_c(gr)
        for c in range(C):
            assert np.linalg.norm(gg[c] - gref[c]) / np.linalg.norm(gref[c]) <= 1e-5


def test_synthesised_channel_end_to_end(cuda_device):
    """f3 feeding the path: synthesise, load, apply; output vs the oracle convolution
    of the oracle-synthesised snapshots (both tolerances compose)."""
    import torch

    from paper_2601_08217_b200 import Channel, synth_jakes

    rng = np.random.default_rng(8)
    C, P, S, N = 4, 10, 256, 20_000
    K = (N - 1) // S + 2
    tau = np.sort(rng.uniform(0, 500, (C, P)), axis=1).astype(np.float32)
    pw = np.exp(-3 * tau / 500).astype(np.float32)
    pw /= pw.sum(axis=1, keepdims=True)
    d, g = synth_jakes(tau, pw, 32, 0.01, seed=5, first_index=0, count=K, device=cuda_device)
    dr, gr = oracle.synth_jakes(tau, pw, 32, 0.01, 5, 0, K)
    x = ttsynth.iq(ttsynth.get("c4").scaled(ues=C, dirs=1, n_per_call=N), 0, C, 0)
    with Channel(d, S, seed=1, snapshot_capacity=K, device=cuda_device) as ch:
        ch.load_snapshots(g, 0)
        y = ch.apply(torch.from_numpy(x).to(cuda_device)).cpu().numpy()
    ref = oracle.convolve(dr, S, gr, 0, x, 0, 0, N)
    compare(y, ref, "synthesised channel")


def test_random_next_instances(cuda_device):
    """Property sweep over the NEXT rows: random shapes, snapshot periods, noise and
    call splits for f1 group sums (random G dividing C) and f2 top-n taps; each against
    the oracle, streamed == one-shot bit for bit. TT_FUZZ_INSTANCES / TT_FUZZ_SEED widen
    it for stress runs."""
    import os

    import torch

    from paper_2601_08217_b200 import Channel

    rng = np.random.default_rng(int(os.environ.get("TT_FUZZ_SEED", "2027")))
    for inst in range(int(os.environ.get("TT_FUZZ_INSTANCES", "20"))):
        G = int(rng.integers(1, 20))
        C = G * int(rng.integers(1, 4))
        L = int(rng.integers(2, 60))
        D = int(rng.integers(L - 1, 4 * L + 50))
        S = int(rng.choice([16, 64, 100, 128, 256, 512]))
        N = int(rng.integers(1, 12_001))
        sigma = float(rng.choice([0.0, 0.05]))
        top_n = int(rng.integers(1, L))
        d = np.stack([np.sort(rng.choice(D + 1, L, replace=False)) for _ in range(C)]).astype(np.int32)
        K = (N - 1) // S + 2
        g = (rng.standard_normal((C, K, L, 2)) / np.sqrt(2 * L)).astype(np.float32)
        x = (rng.standard_normal((C, N, 2)) * np.sqrt(0.5)).astype(np.float32)
        cut = int(rng.integers(1, N)) if N > 1 else N
        splits = ([cut, N - cut] if N > 1 else [N], [N])
        gd = torch.from_numpy(g).to(cuda_device)
        aggs, ys_sparse = [], []
        for split in splits:
            ch = Channel(d, S, seed=inst, snapshot_capacity=K, device=cuda_device)
            ch.load_snapshots(gd, 0)
            a, pos = [], 0
            for n in split:
                a.append(ch.apply_aggregate(torch.from_numpy(np.ascontiguousarray(x[:, pos:pos + n])).to(cuda_device),
                                            G, noise_sigma=sigma).cpu().numpy())
                pos += n
            ch.close()
            aggs.append(np.concatenate(a, axis=1))
            ch = Channel(d, S, seed=inst, snapshot_capacity=K, device=cuda_device)
            ch.set_top_n(top_n)
            ch.load_snapshots(gd, 0)
            yv, pos = [], 0
            for n in split:
                yv.append(ch.apply(torch.from_numpy(np.ascontiguousarray(x[:, pos:pos + n])).to(cuda_device),
                                   noise_sigma=sigma).cpu().numpy())
                pos += n
            ch.close()
            ys_sparse.append(np.concatenate(yv, axis=1))
        what = f"instance {inst}: G={G} C={C} L={L} D={D} S={S} N={N} top_n={top_n}"
        assert np.array_equal(aggs[0], aggs[1]) and np.array_equal(ys_sparse[0], ys_sparse[1]), what
        ref = oracle.convolve(d, S, g, 0, x, 0, 0, N, sigma=sigma, seed=inst)
        compare(aggs[0], oracle.aggregate(ref, G), "agg " + what)
        ref_s = oracle.convolve(d, S, g, 0, x, 0, 0, N, sigma=sigma, seed=inst, top_n=top_n)
        compare(ys_sparse[0], ref_s, "sparse " + what)
