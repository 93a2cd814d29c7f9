"""Parity of the CUDA path (through the C ABI) with the oracle on the same seeded
inputs: every BASELINE config (scaled to oracle-friendly sizes that still span many
tiles and a ragged tail), closed-form special cases bit-exactly, streaming /
isolation / sharding invariances, the bit-exact noise, the generic kernel, the
host-buffer path, and error codes."""
import numpy as np
import pytest

import oracle
import ttsynth
from harness import Run, compare, to_c

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,kw", [
    ("c1", {}),                                                        # full size
    ("c2", dict(n_per_call=300_001)),                                  # ragged tail, noise
    ("c3", dict(ues=4, calls=3)),                                      # streaming slots, DL+UL
    ("c4", dict(ues=3, calls=3)),
    ("c5-L1", dict(ues=4, n_per_call=100_003)),
    ("c5-L4", dict(ues=4, n_per_call=100_003)),
    ("c5-L16", dict(ues=4, n_per_call=100_003)),
    ("c5-L64", dict(ues=2, n_per_call=65_537)),
    ("c5-L256", dict(ues=2, n_per_call=40_001)),
])
def test_config_parity(cuda_device, name, kw):
    w = ttsynth.get(name).scaled(**kw)
    run = Run(w, seed=1234)
    y = run.gpu(cuda_device)
    compare(y, run.oracle(), name)


def test_identity_bit_exact(cuda_device):
    """L=1, d=0, g == 1 -> y == x bit for bit (fma(a, 0, 1) = 1; the cross term is 0)."""
    w = ttsynth.get("c1").scaled(fixed_delays=(0,), fixed_pdp=(1.0,), L=1, D=0, S=64, n_per_call=10_001)
    run = Run(w)
    run.gains[...] = 0.0
    run.gains[..., 0] = 1.0
    y = run.gpu(cuda_device)
    assert np.array_equal(y, run.x)


def test_pure_delay_bit_exact(cuda_device):
    D = 777
    w = ttsynth.get("c1").scaled(fixed_delays=(D,), fixed_pdp=(1.0,), L=1, D=D, S=100, n_per_call=5_000, calls=3)
    run = Run(w)
    run.gains[...] = 0.0
    run.gains[..., 0] = 1.0
    y = run.gpu(cuda_device, calls=[100, 4_000, 10_900])
    assert np.all(y[:, :D] == 0)
    assert np.array_equal(y[:, D:], run.x[:, :-D])


def test_streaming_bit_identical_any_partition(cuda_device):
    """slot-streamed output with carried history == one-shot, here bit for bit,
    for partitions with n < H, odd n, and n not a multiple of anything."""
    w = ttsynth.get("c4").scaled(ues=2, n_per_call=20_000, calls=1)
    run = Run(w, seed=5)
    one = run.gpu(cuda_device, calls=[20_000])
    for calls in ([1, 2, 3, 1000, 1023, 17_971], [999, 5, 18_996], [7_001, 7_001, 5_998], [4_096] * 4 + [3_616]):
        y = run.gpu(cuda_device, calls=calls)
        assert np.array_equal(y, one), calls
    compare(one, run.oracle(), "c4 scaled")


def test_isolation(cuda_device):
    """S:357 / P:23 per-UE isolation: changing channel 1's taps leaves channel 0 and 2
    bit-identical."""
    w = ttsynth.get("c3").scaled(ues=2, dirs=1, n_per_call=9_000, calls=2)
    a = Run(w, seed=3)
    b = Run(w, seed=3)
    b.gains[1] *= -0.5
    b.gains[1, :, 0] += 0.25
    ya, yb = a.gpu(cuda_device), b.gpu(cuda_device)
    assert np.array_equal(ya[0], yb[0])
    assert not np.array_equal(ya[1], yb[1])


def test_sharding_invariance(cuda_device):
    """Two handles over channel blocks with global channel offsets == one handle."""
    w = ttsynth.get("c3").scaled(ues=6, n_per_call=5_000, calls=2)
    full = Run(w, seed=11).gpu(cuda_device)
    for lo, hi in ((0, 4), (4, 10), (10, 12)):
        part = Run(w, lo, hi, seed=11).gpu(cuda_device)
        assert np.array_equal(part, full[lo:hi]), (lo, hi)


def test_noise_bit_exact(cuda_device):
    """x == 0 -> y == w; GPU noise equals the oracle's bit for bit, for even and odd
    call starts (both Philox sharing paths)."""
    w = ttsynth.get("c2").scaled(ues=3, n_per_call=12_345, calls=1)
    run = Run(w, seed=0xDEADBEEF12345)
    run.x[...] = 0.0
    y = run.gpu(cuda_device, calls=[1, 6_000, 6_344])
    for c in range(run.C):
        ref = oracle.noise_block(run.seed, c, 0, run.N, run.sigma)
        assert np.array_equal(y[c], ref), c


def test_generic_kernel_path(cuda_device):
    """A plan that does not fit shared memory (long filter, S = 1) takes the generic
    kernel; it matches the oracle and the streaming invariance still holds."""
    rng = np.random.default_rng(0)
    L = 1500
    w = ttsynth.get("c2").scaled(ues=2, L=L, D=3000, S=1, n_per_call=3_001, snr_db=10.0)
    run = Run(w, seed=2)
    y1 = run.gpu(cuda_device)
    y2 = run.gpu(cuda_device, calls=[1_000, 2_001])
    assert np.array_equal(y1, y2)
    compare(y1, run.oracle(), "generic")


def test_host_buffer_path_equals_device_path(cuda_device):
    w = ttsynth.get("c3").scaled(ues=5, n_per_call=7_000, calls=2)
    run = Run(w, seed=4)
    assert np.array_equal(run.gpu(cuda_device, host_path=True), run.gpu(cuda_device))


def test_host_buffer_path_many_chunks(cuda_device, monkeypatch):
    """128 channels in 1 MiB chunks (32 channels each): the host path cycles its four
    staging buffers and both copy-stream pairs; equal to the device path bit for bit."""
    monkeypatch.setenv("TT_HOST_CHUNK_MB", "1")
    w = ttsynth.get("c3").scaled(ues=64, n_per_call=4_096, calls=2)
    run = Run(w, seed=8)
    assert np.array_equal(run.gpu(cuda_device, host_path=True), run.gpu(cuda_device))


def test_snapshot_ring_streaming(cuda_device):
    """A ring smaller than the run, refilled slot by slot (as a streaming user would)."""
    import torch

    from paper_2601_08217_b200 import Channel

    w = ttsynth.get("c4").scaled(ues=2, calls=4)
    run = Run(w, seed=8)
    ref = run.gpu(cuda_device)
    per = w.n_per_call // w.S
    ch = Channel(run.delays, w.S, seed=8, snapshot_capacity=per + 2, device=cuda_device)
    g = torch.from_numpy(run.gains).to(cuda_device)
    out = []
    for s in range(w.calls):
        lo = s * per
        hi = min(run.K, (s + 1) * per + 2)
        ch.load_snapshots(g[:, lo:hi].contiguous(), lo)
        xs = torch.from_numpy(np.ascontiguousarray(run.x[:, s * w.n_per_call:(s + 1) * w.n_per_call])).to(cuda_device)
        out.append(ch.apply(xs, noise_sigma=run.sigma).cpu().numpy())
    ch.close()
    assert np.array_equal(np.concatenate(out, axis=1), ref)


def test_error_codes(cuda_device):
    import torch

    from paper_2601_08217_b200 import Channel, TTError

    ch = Channel([[0, 3]], 16, snapshot_capacity=4, device=cuda_device)
    x = torch.zeros((1, 64, 2), device=cuda_device)
    with pytest.raises(TTError, match="SNAPSHOT_MISSING"):
        ch.apply(x)
    ch.load_snapshots(torch.zeros((1, 4, 2, 2), device=cuda_device), 0)  # k = 0..3 -> n < 48
    ch.apply(x[:, :47])
    with pytest.raises(TTError, match="SNAPSHOT_MISSING"):
        ch.apply(x[:, :2])  # needs k = 3 and 4
    with pytest.raises(TTError, match="INVALID_ARG"):
        ch.apply(x, out=x)
    with pytest.raises(TTError, match="INVALID_ARG"):
        ch.apply(x[:, :1], noise_sigma=-1.0)
    assert ch.t == 47  # failed calls do not advance the stream
    ch.close()


@pytest.mark.parametrize("name,kw,calls", [
    ("c4", dict(ues=2, n_per_call=20_000, calls=1), [20_000]),
    ("c4", dict(ues=2, n_per_call=20_000, calls=1), [1, 15, 16, 17, 4_095, 4_097, 11_759]),  # 16-misaligned starts
    ("c3", dict(ues=3, n_per_call=9_001, calls=1), [9_001]),
    ("c5-L256", dict(ues=2, n_per_call=9_000), [3_000, 6_000]),
    ("c5-L1", dict(ues=3, n_per_call=5_003), [5_003]),
    ("c1", dict(n_per_call=7_777), [7_777]),
    ("c4", dict(ues=1, n_per_call=12_288, calls=1, S=128), [12_288]),       # 2 intervals per warp
    ("c4", dict(ues=1, n_per_call=12_288, calls=1, S=64), [4_096, 8_192]),  # 4 per warp
    ("c4", dict(ues=1, n_per_call=12_288, calls=1, S=32), [12_288]),        # 8 per warp
    ("c4", dict(ues=1, n_per_call=12_000, calls=1, S=64), [100, 11_900]),   # warps off interval starts
])
def test_kernels_bit_identical(cuda_device, monkeypatch, name, kw, calls):
    """The tiled kernel (default), its robust variant (lead-in tile and window shift, used
    for calls that do not start on a 32R-aligned sample or rows off a 16-B boundary; forced
    here with TT_ROBUST=1), the register-window kernels and the generic kernel run the
    same per-output operation sequence: outputs are equal bit for bit, for any call split
    (history carried across 16-misaligned call starts). The dense-window kernel (forced
    with TT_KERNEL=dw) runs the calls that start and end on 16-sample multiples and hands
    the delay line to and from the tiled kernel for the others."""
    w = ttsynth.get(name).scaled(**kw)
    run = Run(w, seed=21)
    outs = {}
    for k in ("rw", "rw8", "tiled", "generic", "dw"):
        monkeypatch.setenv("TT_KERNEL", k)
        outs[k] = run.gpu(cuda_device, calls=calls)
    monkeypatch.setenv("TT_KERNEL", "tiled")
    monkeypatch.setenv("TT_ROBUST", "1")
    outs["robust"] = run.gpu(cuda_device, calls=calls)
    monkeypatch.delenv("TT_ROBUST")
    monkeypatch.delenv("TT_KERNEL")
    assert np.array_equal(outs["robust"], outs["tiled"])
    assert np.array_equal(outs["rw"], outs["tiled"])
    assert np.array_equal(outs["rw8"], outs["tiled"])
    assert np.array_equal(outs["rw"], outs["generic"])
    assert np.array_equal(outs["dw"], outs["tiled"])
    compare(outs["rw"], run.oracle(), name)


@pytest.mark.parametrize("case", ["max_delay", "many_taps", "max_taps", "duplicate_delays", "one_sample_calls",
                                  "unaligned_rows"])
def test_edge_cases(cuda_device, case):
    """Edge cases of the boundary: the largest delay (TT_MAX_DELAY), very many taps and
    the largest tap count (TT_MAX_TAPS), every tap at the same delay (duplicates add),
    1-sample calls (every call shorter than the delay line), and input / output rows
    that start 8 B off a 16-B boundary (the TMA staging splits off an 8-B head)."""
    import torch

    from paper_2601_08217_b200 import Channel

    if case == "max_delay":
        w = ttsynth.get("c1").scaled(fixed_delays=(0, 4096), fixed_pdp=(0.5, 0.5), L=2, D=4096, S=64,
                                     n_per_call=9_001)
        calls = [5_000, 4_001]
    elif case == "many_taps":
        w = ttsynth.get("c2").scaled(ues=1, L=2000, D=4000, S=512, n_per_call=6_000, snr_db=10.0)
        calls = [6_000]
    elif case == "max_taps":
        w = ttsynth.get("c2").scaled(ues=1, L=4096, D=4096, S=256, n_per_call=1_500, snr_db=10.0)
        calls = [700, 800]
    elif case == "duplicate_delays":
        w = ttsynth.get("c1").scaled(fixed_delays=(5,) * 8, fixed_pdp=(0.125,) * 8, L=8, D=5, S=100,
                                     n_per_call=3_001)
        calls = [1_000, 2_001]
    elif case == "one_sample_calls":
        w = ttsynth.get("c3").scaled(ues=1, dirs=2, n_per_call=40, calls=1)
        calls = [1] * 40
    else:
        w = ttsynth.get("c4").scaled(ues=2, n_per_call=5_001, calls=1)
        calls = [5_001]
    run = Run(w, seed=23)
    if case != "unaligned_rows":
        y = run.gpu(cuda_device, calls=calls)
    else:
        ch = Channel(run.delays, w.S, seed=23, snapshot_capacity=run.K, device=cuda_device)
        ch.load_snapshots(torch.from_numpy(run.gains).to(cuda_device), 0)
        n = calls[0]
        big_x = torch.zeros((run.C * n + 1) * 2, dtype=torch.float32, device=cuda_device)
        big_y = torch.zeros_like(big_x)
        xs = big_x[2:].view(run.C, n, 2)  # 8 B past a 16-B boundary
        xs.copy_(torch.from_numpy(run.x).to(cuda_device))
        ys = big_y[2:].view(run.C, n, 2)
        assert xs.data_ptr() % 16 == 8 and ys.data_ptr() % 16 == 8
        ch.apply(xs, out=ys, noise_sigma=run.sigma)
        torch.cuda.synchronize()
        y = ys.cpu().numpy()
        ch.close()
        assert np.array_equal(y, run.gpu(cuda_device))
    compare(y, run.oracle(), case)


def test_minimal_snapshot_capacity_streaming(cuda_device):
    """snapshot_capacity = 2 (the minimum): each call covers one snapshot interval and the
    next snapshot is loaded just before it, so the ring wraps every call; the streamed
    output equals the oracle on the whole gain sequence."""
    import torch

    from paper_2601_08217_b200 import Channel

    w = ttsynth.get("c4").scaled(ues=2, n_per_call=512, calls=8, S=512)
    run = Run(w, seed=31)
    assert run.K >= w.calls + 1
    ch = Channel(run.delays, w.S, seed=run.seed, snapshot_capacity=2, device=cuda_device)
    try:
        ch.load_snapshots(torch.from_numpy(np.ascontiguousarray(run.gains[:, 0:2])).to(cuda_device), 0)
        ys = []
        for k in range(w.calls):
            if k > 0:
                ch.load_snapshots(torch.from_numpy(np.ascontiguousarray(run.gains[:, k + 1:k + 2])).to(cuda_device),
                                  k + 1)
            info = ch.info()
            assert (info.resident_lo, info.resident_hi) == (k, k + 2)
            xs = torch.from_numpy(np.ascontiguousarray(run.x[:, k * 512:(k + 1) * 512])).to(cuda_device)
            ys.append(ch.apply(xs, noise_sigma=run.sigma).cpu().numpy())
    finally:
        ch.close()
    compare(np.concatenate(ys, axis=1), run.oracle(), "capacity 2")


def test_random_instances_vs_oracle(cuda_device):
    """SPEC AC1-style property sweep: many random instances — channel count,
    taps, delay span, snapshot period (powers of two and not), noise on/off, random
    call splits (streamed == one-shot) — each against the oracle. Covers every plan
    the library picks (tiled R = 8/4/2 with fast / grouped / per-row gain paths, and
    the generic kernel)."""
    import torch

    from paper_2601_08217_b200 import Channel

    import os

    # TT_FUZZ_INSTANCES / TT_FUZZ_SEED / TT_FUZZ_MAX_N widen the sweep for stress runs
    rng = np.random.default_rng(int(os.environ.get("TT_FUZZ_SEED", "2026")))
    max_n = int(os.environ.get("TT_FUZZ_MAX_N", "4096"))
    kinds = set()
    for inst in range(int(os.environ.get("TT_FUZZ_INSTANCES", "60"))):
        C = int(rng.integers(1, 6))
        L = int(rng.integers(1, 101))
        D = int(rng.integers(L - 1, 4 * L + 50)) if L > 1 else int(rng.integers(0, 50))
        S = int(rng.choice([1, 3, 16, 32, 64, 100, 128, 256, 333, 512, 1024]))
        N = int(rng.integers(1, max_n + 1))
        sigma = float(rng.choice([0.0, 0.05]))
        d = np.stack([np.sort(rng.choice(D + 1, L, replace=D + 1 < L)) for _ in range(C)]).astype(np.int32)
        K = (N - 1) // S + 2
        g = (rng.standard_normal((C, K, L, 2)) / np.sqrt(2 * L)).astype(np.float32)
        x = (rng.standard_normal((C, N, 2)) * np.sqrt(0.5)).astype(np.float32)
        cuts = np.sort(rng.choice(np.arange(1, N), size=min(int(rng.integers(0, 4)), N - 1), replace=False)) \
            if N > 1 else np.array([], int)
        calls = np.diff(np.concatenate([[0], cuts, [N]])).astype(int)
        outs = []
        for split in (calls, [N]):
            ch = Channel(d, S, seed=inst, snapshot_capacity=K, device=cuda_device)
            kinds.add(int(ch.info().kernel) * 100 + int(ch.info().outputs_per_thread))
            ch.load_snapshots(torch.from_numpy(g).to(cuda_device), 0)
            ys, pos = [], 0
            for n in split:
                ys.append(ch.apply(torch.from_numpy(np.ascontiguousarray(x[:, pos:pos + n])).to(cuda_device),
                                   noise_sigma=sigma).cpu().numpy())
                pos += int(n)
            ch.close()
            outs.append(np.concatenate(ys, axis=1))
        assert np.array_equal(outs[0], outs[1]), (inst, C, L, D, S, N, list(calls))
        ref = oracle.convolve(d, S, g, 0, x, 0, 0, N, sigma=sigma, seed=inst)
        if np.abs(ref).max() > 0:
            compare(outs[0], ref, f"instance {inst}: C={C} L={L} D={D} S={S} N={N}")
    assert len(kinds) >= 3, kinds  # several plans were exercised


def test_device_clock_cuda_graph_replay(cuda_device):
    """slot calls captured into a CUDA graph replay the next slots
    (device-clock mode: t and the delay-line half live on the GPU), bit-identical to
    eager calls, and the clock reads back into the handle."""
    import torch

    from paper_2601_08217_b200 import Channel, TTError

    n, calls, per_graph = 4_096, 6, 2
    w = ttsynth.get("c4").scaled(ues=3, n_per_call=n, calls=calls)
    run = Run(w, seed=77)
    eager = run.gpu(cuda_device)
    compare(eager, run.oracle(), "device clock (eager reference)")

    ch = Channel(run.delays, w.S, seed=run.seed, snapshot_capacity=run.K, device=cuda_device)
    try:
        ch.load_snapshots(torch.from_numpy(run.gains).to(cuda_device), 0)
        ch.set_device_clock(True)
        assert ch.info().device_clock == 1
        xs = [torch.zeros((run.C, n, 2), dtype=torch.float32, device=cuda_device) for _ in range(per_graph)]
        ys = [torch.zeros_like(x) for x in xs]
        with pytest.raises(TTError, match="UNSUPPORTED"):
            ch.apply(xs[0][:, :100].contiguous(), noise_sigma=run.sigma)  # n % 256 != 0
        with pytest.raises(TTError, match="UNSUPPORTED"):
            ch.set_top_n(2)  # could re-plan away from the tiled kernel
        xh = xs[0].cpu().pin_memory()
        with pytest.raises(TTError, match="UNSUPPORTED"):
            ch.apply_host(xh, torch.empty_like(xh).pin_memory(), noise_sigma=run.sigma)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for k in range(per_graph):
                ch.apply(xs[k], out=ys[k], noise_sigma=run.sigma)
        out = np.empty_like(eager)
        for r in range(calls // per_graph):
            for k in range(per_graph):
                c = r * per_graph + k
                xs[k].copy_(torch.from_numpy(np.ascontiguousarray(run.x[:, c * n:(c + 1) * n])))
            g.replay()
            torch.cuda.synchronize()
            for k in range(per_graph):
                c = r * per_graph + k
                out[:, c * n:(c + 1) * n] = ys[k].cpu().numpy()
        assert np.array_equal(out, eager)
        ch.set_device_clock(False)
        assert ch.t == calls * n and ch.info().device_clock == 0
    finally:
        ch.close()
    # entering the mode off the 256-sample grid is refused
    ch = Channel(run.delays, w.S, seed=run.seed, snapshot_capacity=run.K, device=cuda_device)
    try:
        ch.load_snapshots(torch.from_numpy(run.gains).to(cuda_device), 0)
        ch.apply(torch.zeros((run.C, 100, 2), dtype=torch.float32, device=cuda_device), noise_sigma=run.sigma)
        with pytest.raises(TTError, match="UNSUPPORTED"):
            ch.set_device_clock(True)
    finally:
        ch.close()


def test_device_clock_graph_aggregate(cuda_device):
    """apply_aggregate captured in a CUDA graph (one uncaptured call first allocates its
    scratch): the replays give the same group sums as eager calls."""
    import torch

    from paper_2601_08217_b200 import Channel

    n, calls, G = 2_048, 4, 8
    w = ttsynth.get("c4").scaled(ues=8, dirs=2, n_per_call=n, calls=calls + 1)
    run = Run(w, seed=78)
    xs_all = torch.from_numpy(run.x).to(cuda_device)
    g_dev = torch.from_numpy(run.gains).to(cuda_device)

    def eager():
        ch = Channel(run.delays, w.S, seed=run.seed, snapshot_capacity=run.K, device=cuda_device)
        ch.load_snapshots(g_dev, 0)
        outs = [ch.apply_aggregate(xs_all[:, c * n:(c + 1) * n].contiguous(), G, noise_sigma=run.sigma).cpu()
                for c in range(calls + 1)]
        ch.close()
        return torch.cat(outs, dim=1).numpy()

    ref = eager()
    ch = Channel(run.delays, w.S, seed=run.seed, snapshot_capacity=run.K, device=cuda_device)
    try:
        ch.load_snapshots(g_dev, 0)
        x0 = xs_all[:, :n].contiguous()
        agg0 = ch.apply_aggregate(x0, G, noise_sigma=run.sigma)  # uncaptured: allocates the scratch
        ch.set_device_clock(True)
        xin = torch.empty_like(x0)
        agg = torch.empty_like(agg0)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            ch.apply_aggregate(xin, G, agg=agg, noise_sigma=run.sigma)
        got = [agg0.cpu()]
        for c in range(1, calls + 1):
            xin.copy_(xs_all[:, c * n:(c + 1) * n])
            g.replay()
            got.append(agg.cpu())
        ch.set_device_clock(False)
        assert np.array_equal(torch.cat(got, dim=1).numpy(), ref)
    finally:
        ch.close()
