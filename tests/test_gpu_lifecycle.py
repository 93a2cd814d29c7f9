"""Handle-lifecycle regressions on the GPU, through the C ABI (round-2 review items):

* clearing an input map while sparse top-n is on must not touch the sparse ring;
* a second handle with a smaller shared-memory plan must not break a live handle
  (the max-dynamic-smem attribute is process-wide, per kernel function);
* reloading snapshots strictly inside the resident range recomputes the differences
  to both resident neighbours (the interpolation through the reloaded block uses the
  new values on both sides);
* the torch wrapper refuses tensors on the wrong device or of the wrong dtype;
* a failed set_top_n leaves the handle dense with a dense plan;
* host-memory snapshot loads on different streams do not race on the staging buffer.

Every output is compared with the oracle on the same seeded inputs."""
import numpy as np
import pytest

import oracle
import ttsynth
from harness import Run, compare

pytestmark = pytest.mark.gpu


def _apply_all(ch, run, device, calls=None):
    import torch

    calls = calls or [run.N]
    out, pos = [], 0
    for n in calls:
        xs = torch.from_numpy(np.ascontiguousarray(run.x[:, pos:pos + n])).to(device)
        out.append(ch.apply(xs, noise_sigma=run.sigma).cpu().numpy())
        pos += n
    torch.cuda.synchronize()
    return np.concatenate(out, axis=1)


class _Poison:
    """cudaMalloc blocks of the given sizes filled with 0xFF bytes (NaN as float32),
    straight from the CUDA runtime (not torch's caching allocator), so that memory a
    library call wrongly freed is likely handed out again and overwritten."""

    def __init__(self, sizes):
        import ctypes

        self.rt = ctypes.CDLL("libcudart.so.12")
        self.ptrs = []
        for nb in sizes:
            p = ctypes.c_void_p()
            if self.rt.cudaMalloc(ctypes.byref(p), ctypes.c_size_t(nb)) == 0:
                self.rt.cudaMemset(p, 0xFF, ctypes.c_size_t(nb))
                self.ptrs.append(p)
        self.rt.cudaDeviceSynchronize()

    def free(self):
        for p in self.ptrs:
            self.rt.cudaFree(p)
        self.ptrs = []


def test_clear_input_map_keeps_sparse_ring(cuda_device):
    """set_top_n(k) -> set_input_map(rows) -> set_input_map(None) -> apply: the
    sparse result still matches the oracle (the map never owned the sparse ring).
    Blocks of the sparse ring's sizes are allocated and poisoned in between, so a
    ring freed by mistake may be overwritten with NaN (best effort: the driver does
    not promise to hand a freed range out again, and on the round-1 library this
    test still passed — the fix is checked by the code path, this guards the result)."""
    import torch

    from paper_2601_08217_b200 import Channel

    w = ttsynth.get("c4").scaled(ues=2, n_per_call=9_000, calls=1)
    run = Run(w, seed=21)
    top_n = 12
    n4 = (top_n + 1 + 3) & ~3
    cap = 1 << 16  # a large ring: tens of MB, whose freed address range the driver reuses
    ch = Channel(run.delays, w.S, seed=run.seed, snapshot_capacity=cap, device=cuda_device)
    poison = None
    try:
        ch.set_top_n(top_n)
        ch.load_snapshots(torch.from_numpy(run.gains).to(cuda_device), 0)
        ch.set_input_map(np.arange(run.C, dtype=np.int32)[::-1].copy(), run.C)
        ch.set_input_map(None)
        poison = _Poison([(run.C * cap * top_n + 1) * 16, run.C * cap * n4 * 4] * 2)
        assert ch.info().top_n == top_n
        y = _apply_all(ch, run, cuda_device, [4_000, 5_000])
        # the next load selects into the same sparse ring (a freed ring would fault here)
        ch.load_snapshots(torch.from_numpy(run.gains).to(cuda_device), 0)
        torch.cuda.synchronize()
    finally:
        ch.close()
        if poison is not None:
            poison.free()
    ref = oracle.convolve(run.delays, w.S, run.gains, 0, run.x, 0, 0, run.N, sigma=run.sigma, seed=run.seed,
                          top_n=top_n)
    compare(y, ref, "sparse after clearing the input map")


def test_second_handle_with_smaller_plan_keeps_first_working(cuda_device):
    """A c4-shaped handle (large shared-memory plan), then a c3-shaped one with a
    smaller plan created after it: both apply correctly, in either order."""
    import torch

    from paper_2601_08217_b200 import Channel

    runs = [Run(ttsynth.get("c4").scaled(ues=2, n_per_call=8_192, calls=1), seed=3),
            Run(ttsynth.get("c3").scaled(ues=2, n_per_call=6_000, calls=1), seed=4),
            Run(ttsynth.get("c5-L1").scaled(ues=2, n_per_call=5_000), seed=5)]
    chans = []
    try:
        for r in runs:
            ch = Channel(r.delays, r.w.S, seed=r.seed, snapshot_capacity=r.K, device=cuda_device)
            ch.load_snapshots(torch.from_numpy(r.gains).to(cuda_device), 0)
            chans.append(ch)
        outs = [None] * len(runs)
        for i in (0, 2, 1):  # the first (largest plan) handle applies after the smaller ones exist
            outs[i] = _apply_all(chans[i], runs[i], cuda_device)
    finally:
        for ch in chans:
            ch.close()
    for r, y in zip(runs, outs):
        compare(y, r.oracle(), f"handle S={r.w.S} L={r.w.L}")


@pytest.mark.parametrize("top_n", [0, 10])
@pytest.mark.parametrize("block", [(1, 2), (3, 6), (0, 1)])
def test_reload_inside_resident_range(cuda_device, top_n, block):
    """Reload snapshots [lo, hi) strictly inside the resident window with new values:
    the output equals the oracle on the gains with that block replaced — including the
    intervals (lo-1, lo) and (hi-1, hi) that straddle the block's ends."""
    import torch

    from paper_2601_08217_b200 import Channel

    w = ttsynth.get("c4").scaled(ues=2, n_per_call=2_400, calls=1)  # S = 256 -> K = 11 snapshots
    run = Run(w, seed=9)
    lo, hi = block
    rng = np.random.default_rng(1234 + lo)
    new = rng.standard_normal((run.C, hi - lo, w.L, 2)).astype(np.float32) * 0.3
    ch = Channel(run.delays, w.S, seed=run.seed, snapshot_capacity=run.K + 2, device=cuda_device)
    try:
        if top_n:
            ch.set_top_n(top_n)
        ch.load_snapshots(torch.from_numpy(run.gains).to(cuda_device), 0)
        ch.load_snapshots(torch.from_numpy(new).to(cuda_device), lo)
        info = ch.info()
        assert (info.resident_lo, info.resident_hi) == (0, run.K)
        y = _apply_all(ch, run, cuda_device)
    finally:
        ch.close()
    g = run.gains.copy()
    g[:, lo:hi] = new
    ref = oracle.convolve(run.delays, w.S, g, 0, run.x, 0, 0, run.N, sigma=run.sigma, seed=run.seed, top_n=top_n)
    compare(y, ref, f"reload [{lo},{hi}) top_n={top_n}")


def test_wrapper_refuses_foreign_tensors(cuda_device):
    import torch

    from paper_2601_08217_b200 import Channel

    w = ttsynth.get("c3").scaled(ues=2, dirs=1, n_per_call=1_000, calls=1)
    run = Run(w, seed=1)
    with Channel(run.delays, w.S, seed=run.seed, snapshot_capacity=run.K, device=cuda_device) as ch:
        ch.load_snapshots(torch.from_numpy(run.gains).to(cuda_device), 0)
        xc = torch.from_numpy(run.x)
        with pytest.raises(ValueError, match="must be on"):
            ch.apply(xc)  # CPU tensor
        xd = xc.to(cuda_device)
        with pytest.raises(ValueError, match="must be on"):
            ch.apply(xd, out=torch.empty_like(xc))  # CPU out
        with pytest.raises(ValueError):
            ch.apply_aggregate(xd, 2, agg=torch.empty((1, run.N, 2), dtype=torch.float16, device=cuda_device))
        with pytest.raises(ValueError, match="must be on"):
            ch.apply_aggregate(xd, 2, agg=torch.empty((1, run.N, 2), dtype=torch.float32))
        assert ch.t == 0  # nothing was enqueued
        y = ch.apply(xd, noise_sigma=run.sigma).cpu().numpy()
    compare(y, run.oracle(), "after refused calls")


def test_failed_set_top_n_leaves_a_dense_handle(cuda_device):
    """Make the sparse-ring allocation fail (the dense ring takes most of the free
    memory): the call reports OUT_OF_MEMORY and the handle stays dense, with a dense
    plan, and still matches the dense oracle."""
    import torch

    from paper_2601_08217_b200 import Channel, TTError

    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info(cuda_device)
    w = ttsynth.get("c5-L64").scaled(ues=2, n_per_call=3_000)
    run = Run(w, seed=8)
    C, L = run.C, w.L
    # dense ring C x cap x L x 16 B ~ 70 % of free; sparse ring + offsets for n = L - 1 ~ 85 %
    cap = int(0.70 * free / (C * L * 16))
    ch = Channel(run.delays, w.S, seed=run.seed, snapshot_capacity=cap, device=cuda_device)
    try:
        ch.load_snapshots(torch.from_numpy(run.gains).to(cuda_device), 0)
        with pytest.raises(TTError, match="OUT_OF_MEMORY|CUDA"):
            ch.set_top_n(L - 1)
        assert ch.info().top_n == 0
        y = _apply_all(ch, run, cuda_device)
    finally:
        ch.close()
    torch.cuda.empty_cache()
    compare(y, run.oracle(), "dense after a failed set_top_n")


def test_host_loads_on_two_streams_share_the_staging_buffer(cuda_device):
    """Snapshot loads from host memory go through one device staging buffer per handle.
    Blocks loaded from host tensors on two streams back to back, with no host sync in
    between: the second block's copy into the staging buffer must wait for the first
    block's loader kernel (on the other stream) to have read it. Repeated with blocks of
    decreasing size (the buffer is reused, not regrown)."""
    import torch

    from paper_2601_08217_b200 import Channel

    w = ttsynth.get("c4").scaled(ues=64, n_per_call=4_000, calls=1)  # 128 channels, 48 taps, K = 17
    run = Run(w, seed=21)
    K = run.K
    cuts = [0, 9, 14, K]  # blocks of 9, 5 and 3 snapshots
    s1, s2 = torch.cuda.Stream(cuda_device), torch.cuda.Stream(cuda_device)
    ch = Channel(run.delays, w.S, seed=run.seed, snapshot_capacity=K + 2, device=cuda_device)
    try:
        # a first, larger host load sizes the staging buffer for the blocks below
        ch.load_snapshots(torch.zeros(run.C, K, w.L, 2), 0, stream=s1)
        torch.cuda.synchronize()
        for i in range(len(cuts) - 1):
            blk = torch.from_numpy(np.ascontiguousarray(run.gains[:, cuts[i]:cuts[i + 1]]))  # CPU tensor: no wrapper sync
            ch.load_snapshots(blk, cuts[i], stream=s1 if i % 2 == 0 else s2)
        torch.cuda.synchronize()
        y = _apply_all(ch, run, cuda_device)
    finally:
        ch.close()
    ref = oracle.convolve(run.delays, w.S, run.gains, 0, run.x, 0, 0, run.N, sigma=run.sigma, seed=run.seed)
    compare(y, ref, "host loads on two streams")
