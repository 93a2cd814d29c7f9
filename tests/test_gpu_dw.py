"""The dense-window kernel (tt_conv_dw.cuh, TT_KERNEL_DW; opt-in with TT_KERNEL=dw) on the
GPU, through the C ABI.

It runs the per-output operation sequence of the tiled kernel (h = fma(alpha, dg, g),
A += h.re x, B += h.im x over the taps in ascending delay order), so its outputs must
equal the tiled kernel's bit for bit, on every shape it can plan, with and without
noise, for any call split — calls that do not start and end on a multiple of 16 run the
tiled kernel, so the delay line is handed between the two kernels — and match the
oracle within north_star's tolerances."""
import numpy as np
import pytest

import ttsynth
from harness import Run, compare

pytestmark = pytest.mark.gpu

KERNEL_DW, KERNEL_TILED = 3, 1


def _gpu(run, device, calls, kernel=None, monkeypatch=None):
    if kernel is not None:
        monkeypatch.setenv("TT_KERNEL", kernel)
    try:
        return run.gpu(device, calls=calls)
    finally:
        if kernel is not None:
            monkeypatch.delenv("TT_KERNEL")


@pytest.mark.parametrize("name,kw,calls", [
    ("c5-L16", dict(ues=3, n_per_call=20_480), [20_480]),
    ("c5-L16", dict(ues=3, n_per_call=20_480), [4_096, 16, 7_952, 8_416]),    # aligned splits, tail tiles
    ("c5-L16", dict(ues=2, n_per_call=9_000), [1_000, 3_001, 4_999]),         # unaligned: tiled fallback mixed in
    ("c5-L64", dict(ues=2, n_per_call=12_288), [12_288]),
    ("c5-L256", dict(ues=2, n_per_call=6_144), [2_048, 4_096]),               # 4 consumer warps (smem)
    ("c5-L8", dict(ues=2, n_per_call=8_192), [8_192]),
    ("c5-L16", dict(ues=2, n_per_call=8_192, snr_db=10.0), [4_096, 4_096]),  # noise epilogue
    ("c5-L16", dict(ues=2, n_per_call=8_192, S=1024), [8_192]),
    ("c5-L64", dict(ues=2, n_per_call=8_192, S=16), [8_192]),                # many gain rows per tile
    ("c4", dict(ues=2, n_per_call=12_288, calls=1), [12_288]),               # sparse delays (forced dw)
    ("c3", dict(ues=2, n_per_call=8_192, calls=1), [4_096, 4_096]),
    ("c1", dict(n_per_call=4_096), [4_096]),
])
def test_dw_equals_tiled_and_oracle(cuda_device, monkeypatch, name, kw, calls):
    w = ttsynth.get(name).scaled(**kw)
    run = Run(w, seed=41)
    dw = _gpu(run, cuda_device, calls, "dw", monkeypatch)
    tiled = _gpu(run, cuda_device, calls, "tiled", monkeypatch)
    assert np.array_equal(dw, tiled)
    compare(dw, run.oracle(), f"dw {name}")


def test_dw_plan_selection(cuda_device, monkeypatch):
    """The dense-window kernel is opt-in: the default plan is the tiled kernel on every
    BASELINE shape; TT_KERNEL=dw selects it (16 outputs per thread) where it fits."""
    import torch  # noqa: F401

    from paper_2601_08217_b200 import Channel

    for name in ("c5-L16", "c5-L64", "c5-L256", "c4", "c2", "c5-L4"):
        w = ttsynth.get(name).scaled(ues=2, n_per_call=4_096)
        d = ttsynth.delays(w, 0, w.C)
        with Channel(d, w.S, snapshot_capacity=4, device=cuda_device) as ch:
            assert ch.info().kernel == KERNEL_TILED, name
        monkeypatch.setenv("TT_KERNEL", "dw")
        with Channel(d, w.S, snapshot_capacity=4, device=cuda_device) as ch:
            info = ch.info()
            assert info.kernel == KERNEL_DW and info.outputs_per_thread == 16, (name, info.kernel)
        monkeypatch.delenv("TT_KERNEL")


def test_dw_streaming_many_channels_and_sharding(cuda_device):
    """A streamed run over 16-multiple slots with a channel offset (the bench's sharded
    layout): dw == tiled bit for bit, and the oracle agrees."""
    w = ttsynth.get("c5-L16").scaled(ues=40, n_per_call=2_048)
    run = Run(w, c_lo=8, c_hi=40, calls=[2_048, 1_024, 4_096, 512], seed=3)
    import os

    old = os.environ.pop("TT_KERNEL", None)
    try:
        os.environ["TT_KERNEL"] = "dw"
        dw = run.gpu(cuda_device)
        os.environ["TT_KERNEL"] = "tiled"
        tiled = run.gpu(cuda_device)
    finally:
        os.environ.pop("TT_KERNEL", None)
        if old is not None:
            os.environ["TT_KERNEL"] = old
    assert np.array_equal(dw, tiled)
    compare(dw, run.oracle(), "dw streamed, sharded")
