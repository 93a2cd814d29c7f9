"""Row e on the CPU: the N > 1 path with real world_size-2 gloo process groups.

Only one GPU exists in this run, so the multi-rank logic is checked here: the
product's shard rule (`paper_2601_08217_b200.shard`) covers every UE exactly once
with both directions together, agrees with the input generator's rule, and the
per-rank pieces computed with GLOBAL channel ids (noise key, input draws) and
gathered over the process group equal the single-process result bit for bit; the
max / sum reductions bench.py uses behave as the timing rule says."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import ttsynth
from paper_2601_08217_b200 import shard


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, kw, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    try:
        pg = shard.init("gloo")
        assert shard.env() == (rank, world, rank)
        w = ttsynth.get(name).scaled(**kw)
        c_lo, c_hi = shard.ue_block(w.ues, w.dirs, rank, world)
        n = w.n_per_call
        K = (n - 1) // w.S + 2
        d = ttsynth.delays(w, c_lo, c_hi)
        g = ttsynth.snapshots(w, c_lo, c_hi, K)
        x = ttsynth.iq(w, c_lo, c_hi, 0)
        y = oracle.convolve(d, w.S, g, 0, x, 0, 0, n, sigma=w.sigma, seed=77, c_offset=c_lo) if c_hi > c_lo \
            else np.zeros((0, n), np.complex128)
        parts = [None] * world
        dist.all_gather_object(parts, (c_lo, c_hi, y))
        mx = shard.max_over_ranks(10.0 + rank, None, pg)
        sm = shard.sum_over_ranks((c_hi - c_lo) * n, None, pg)
        shard.barrier(pg)
        if rank == 0:
            q.put(("ok", parts, mx, sm))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put(("err", repr(e), None, None))
        raise


@pytest.mark.parametrize("name,kw", [
    ("c4", dict(ues=3, n_per_call=2_000)),           # odd UE count: ranks get 1 and 2 UEs (DL+UL)
    ("c3", dict(ues=1, n_per_call=1_500)),           # fewer UEs than ranks: rank 0 owns nothing
    ("c2", dict(ues=4, n_per_call=3_001)),           # one direction per UE, ragged length
])
def test_two_rank_shards_equal_single_process(name, kw):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, kw, q)) for r in range(world)]
    for p in procs:
        p.start()
    status, parts, mx, sm = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert status == "ok", parts
    assert all(p.exitcode == 0 for p in procs)
    w = ttsynth.get(name).scaled(**kw)
    n = w.n_per_call
    # the blocks tile [0, C) in order, UEs whole
    assert parts[0][0] == 0 and parts[-1][1] == w.C
    for a, b in zip(parts, parts[1:]):
        assert a[1] == b[0]
    for lo, hi, _ in parts:
        assert lo % w.dirs == 0 and hi % w.dirs == 0
    # gathered pieces == one process over all channels (global keys), bit for bit
    K = (n - 1) // w.S + 2
    full = oracle.convolve(ttsynth.delays(w), w.S, ttsynth.snapshots(w, 0, w.C, K), 0, ttsynth.iq(w, 0, w.C, 0), 0, 0,
                           n, sigma=w.sigma, seed=77)
    got = np.concatenate([y for _, _, y in parts], axis=0)
    assert np.array_equal(got, full)
    assert mx == 10.0 + (world - 1)
    assert sm == w.C * n


@pytest.mark.parametrize("ues,dirs,world", [(512, 2, 1), (512, 2, 2), (512, 2, 8), (3, 2, 2), (1, 2, 4), (64, 1, 8)])
def test_ue_block_rule(ues, dirs, world):
    class W:
        pass
    blocks = [shard.ue_block(ues, dirs, r, world) for r in range(world)]
    assert blocks[0][0] == 0 and blocks[-1][1] == ues * dirs
    sizes = [hi - lo for lo, hi in blocks]
    assert max(sizes) - min(sizes) <= dirs  # balanced to within one UE
    w = ttsynth.get("c4").scaled(ues=ues, dirs=dirs)
    assert blocks == [ttsynth.shard_ues(w, r, world) for r in range(world)]
    with pytest.raises(ValueError):
        shard.ue_block(ues, dirs, world, world)


def _agg_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    try:
        pg = shard.init("gloo")
        w = ttsynth.get("c4").scaled(ues=5, dirs=1, n_per_call=1_500, calls=1)  # 5 UL channels, one cell
        c_lo, c_hi = shard.ue_block(w.ues, w.dirs, rank, world)
        n = w.n_per_call
        K = (n - 1) // w.S + 2
        y = oracle.convolve(ttsynth.delays(w, c_lo, c_hi), w.S, ttsynth.snapshots(w, c_lo, c_hi, K), 0,
                            ttsynth.iq(w, c_lo, c_hi, 0), 0, 0, n, sigma=w.sigma, seed=9, c_offset=c_lo)
        part = oracle.aggregate(y, c_hi - c_lo)[0]  # this rank's partial cell sum
        t = torch.from_numpy(np.stack([part.real, part.imag], axis=-1))
        shard.reduce_groups(t, pg)
        if rank == 0:
            q.put(("ok", t.numpy()))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put(("err", repr(e)))
        raise


def test_cell_aggregate_reduced_over_ranks():
    """f1 across ranks: per-rank partial cell sums all-reduced == the single-process
    cell aggregate (summation order differs -> tolerance)."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_agg_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    status, got = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert status == "ok", got
    w = ttsynth.get("c4").scaled(ues=5, dirs=1, n_per_call=1_500, calls=1)
    n = w.n_per_call
    K = (n - 1) // w.S + 2
    full = oracle.aggregate(oracle.convolve(ttsynth.delays(w), w.S, ttsynth.snapshots(w, 0, w.C, K), 0,
                                            ttsynth.iq(w, 0, w.C, 0), 0, 0, n, sigma=w.sigma, seed=9), w.C)[0]
    assert np.allclose(got[:, 0] + 1j * got[:, 1], full, rtol=0, atol=1e-12)
