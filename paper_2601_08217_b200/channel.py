"""`Channel`: a thin torch-facing wrapper over one tt_channel handle.

PyTorch supplies device memory and streams only; every sample is computed by the
library's kernels (see include/tt_channel.h for semantics and errors).
"""
from __future__ import annotations

from typing import Optional

import numpy as np
import torch

from . import _lib


def _stream_ptr(stream: Optional[torch.cuda.Stream], device: Optional[torch.device] = None) -> int:
    """The given stream, else the current stream of `device` (the channel's device,
    not whatever device happens to be current)."""
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return int(s.cuda_stream)


def _check_dev(name: str, t: torch.Tensor, device: torch.device) -> None:
    # a CPU tensor or one on another GPU would reach the kernel as a foreign pointer
    # and fault the context: refuse it here
    if t.device != device:
        raise ValueError(f"{name} must be on {device}, got {t.device}")


class Channel:
    """C = num_ue channel streams with L taps at integer delays (host [C][L])."""

    def __init__(self, delays, snapshot_period: int, seed: int = 0, snapshot_capacity: int = 2,
                 channel_offset: int = 0, device: Optional[torch.device] = None):
        d = np.ascontiguousarray(np.asarray(delays, dtype=np.int32))
        if d.ndim != 2:
            raise ValueError("delays must be [C][L]")
        self.C, self.L = int(d.shape[0]), int(d.shape[1])
        self.S = int(snapshot_period)
        dev = torch.device("cuda") if device is None else torch.device(device)
        if dev.type != "cuda":
            raise ValueError(f"a Channel lives on a CUDA device, got {dev}")
        # an explicit index, so tensor-device checks compare like with like
        self.device = dev if dev.index is not None else torch.device("cuda", torch.cuda.current_device())
        self._h = None
        with torch.cuda.device(self.device):
            self._h = _lib.tt_channel_create(self.C, self.L, d.ctypes.data, self.S, int(seed), int(snapshot_capacity),
                                             int(channel_offset))

    # -- lifecycle -------------------------------------------------------------------
    def close(self) -> None:
        if self._h is not None:
            _lib.tt_channel_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def handle(self) -> int:
        if self._h is None:
            raise RuntimeError("channel is closed")
        return self._h

    def info(self) -> _lib.ChannelInfo:
        return _lib.tt_channel_get_info(self.handle)

    @property
    def t(self) -> int:
        return int(self.info().t)

    # -- calls -----------------------------------------------------------------------
    def load_snapshots(self, gains, first_index: int, stream: Optional[torch.cuda.Stream] = None) -> None:
        """gains: float32 [C][count][L][2] (torch tensor on this device or host, or numpy)."""
        if isinstance(gains, np.ndarray):
            g = np.ascontiguousarray(gains, dtype=np.float32)
            ptr, count = g.ctypes.data, g.shape[1]
            keep = g
        else:
            g = gains.contiguous()
            if g.dtype != torch.float32:
                raise TypeError("gains must be float32")
            ptr, count = g.data_ptr(), g.shape[1]
            keep = g
        if tuple(keep.shape[:1]) != (self.C,) or keep.shape[2:] != (self.L, 2):
            raise ValueError(f"gains must be [C={self.C}][count][L={self.L}][2], got {tuple(keep.shape)}")
        if not isinstance(keep, np.ndarray) and keep.device.type == "cuda":
            _check_dev("gains", keep, self.device)
        _lib.tt_channel_load_snapshots(self.handle, ptr, int(first_index), int(count), _stream_ptr(stream, self.device))
        if isinstance(keep, np.ndarray):
            # host pageable source: make sure the copy has consumed it before returning
            torch.cuda.current_stream(self.device).synchronize() if stream is None else stream.synchronize()

    def apply(self, x: torch.Tensor, out: Optional[torch.Tensor] = None, noise_sigma: float = 0.0,
              stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        """x: float32 device tensor [C][n][2] (or complex64 [C][n]); returns y alike."""
        cplx = x.is_complex()
        xv = torch.view_as_real(x) if cplx else x
        rows = getattr(self, "in_rows", self.C)
        shape = xv.shape
        if xv.dtype != torch.float32 or len(shape) != 3 or shape[0] != rows or shape[2] != 2:
            raise ValueError(f"x must be float32 [{rows}][n][2] or complex64 [{rows}][n]")
        if not xv.is_contiguous():
            raise ValueError("x must be contiguous")
        dev = self.device
        _check_dev("x", xv, dev)
        n = shape[1]
        if out is None:
            out = torch.empty((self.C, n, 2), dtype=torch.float32, device=xv.device)
            if cplx:
                out = torch.view_as_complex(out)
            ov = torch.view_as_real(out) if cplx else out
        else:
            ov = torch.view_as_real(out) if out.is_complex() else out
            oshape = ov.shape
            if len(oshape) != 3 or oshape[0] != self.C or oshape[1] != n or oshape[2] != 2 or \
                    not ov.is_contiguous() or ov.dtype != torch.float32:
                raise ValueError(f"out must be contiguous float32 [C={self.C}][n][2]")
            _check_dev("out", ov, dev)
        h = self._h
        if h is None:
            raise RuntimeError("channel is closed")
        _lib.tt_channel_apply(h, xv.data_ptr(), ov.data_ptr(), n, float(noise_sigma), _stream_ptr(stream, dev))
        return out

    def set_top_n(self, top_n: int) -> None:
        """NEXT f2: sum only the top_n dominant taps per snapshot interval (0 = dense)."""
        _lib.tt_channel_set_top_n(self.handle, int(top_n))

    def set_input_map(self, rows, num_rows: Optional[int] = None) -> None:
        """NEXT f4: channel c reads row rows[c] of the apply input ([num_rows][n][2]);
        None restores the identity."""
        if rows is None:
            _lib.tt_channel_set_input_map(self.handle, None, 0)
            self.in_rows = self.C
            return
        r = np.ascontiguousarray(np.asarray(rows, dtype=np.int32))
        if r.shape != (self.C,):
            raise ValueError(f"rows must have one entry per channel ({self.C})")
        nr = int(r.max()) + 1 if num_rows is None else int(num_rows)
        _lib.tt_channel_set_input_map(self.handle, r.ctypes.data, nr)
        self.in_rows = nr

    def apply_aggregate(self, x: torch.Tensor, group_size: int, agg: Optional[torch.Tensor] = None,
                        out: Optional[torch.Tensor] = None, noise_sigma: float = 0.0,
                        stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        """NEXT f1/f4: apply, and sum the outputs of every group of `group_size`
        consecutive channels: agg [C / group_size][n][2]. `out` ([C][n][2]) optionally
        receives the per-channel outputs."""
        xv = torch.view_as_real(x) if x.is_complex() else x
        rows = getattr(self, "in_rows", self.C)
        if xv.dtype != torch.float32 or xv.dim() != 3 or xv.shape[0] != rows or xv.shape[2] != 2 or \
                not xv.is_contiguous():
            raise ValueError(f"x must be contiguous float32 [{rows}][n][2]")
        _check_dev("x", xv, self.device)
        n = int(xv.shape[1])
        if group_size <= 0 or self.C % group_size:
            raise ValueError(f"group_size must divide C={self.C}")
        if agg is None:
            agg = torch.empty((self.C // group_size, n, 2), dtype=torch.float32, device=xv.device)
        if agg.shape != (self.C // group_size, n, 2) or not agg.is_contiguous() or agg.dtype != torch.float32:
            raise ValueError("agg must be contiguous float32 [C/group_size][n][2]")
        _check_dev("agg", agg, self.device)
        optr = 0
        if out is not None:
            if out.shape != (self.C, n, 2) or not out.is_contiguous() or out.dtype != torch.float32:
                raise ValueError("out must be contiguous float32 [C][n][2]")
            _check_dev("out", out, self.device)
            optr = out.data_ptr()
        _lib.tt_channel_apply_aggregate(self.handle, xv.data_ptr(), optr, agg.data_ptr(), int(group_size), n,
                                        float(noise_sigma), _stream_ptr(stream, self.device))
        return agg

    def apply_host(self, x: torch.Tensor, out: torch.Tensor, noise_sigma: float = 0.0,
                   stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
        """Host tensors (pinned for overlap) [C][n][2]; out is complete when `stream` gets here."""
        if x.device.type != "cpu" or out.device.type != "cpu":
            raise ValueError("apply_host takes host tensors")
        if x.dtype != torch.float32 or x.dim() != 3 or x.shape[0] != self.C or x.shape[2] != 2 or \
                out.shape != x.shape or not (x.is_contiguous() and out.is_contiguous()):
            raise ValueError(f"x, out must be contiguous float32 [C={self.C}][n][2]")
        _lib.tt_channel_apply_host(self.handle, x.data_ptr(), out.data_ptr(), int(x.shape[1]), float(noise_sigma),
                                   _stream_ptr(stream, self.device))
        return out

    def reset(self, stream: Optional[torch.cuda.Stream] = None) -> None:
        _lib.tt_channel_reset(self.handle, _stream_ptr(stream, self.device))

    def set_device_clock(self, enable: bool, stream: Optional[torch.cuda.Stream] = None) -> None:
        """Device-clock mode (tt_channel_set_device_clock): the stream position lives on
        the GPU, so slot calls can be captured into a CUDA graph and replayed; calls
        then need n % 256 == 0 and snapshot residency is the caller's contract."""
        _lib.tt_channel_set_device_clock(self.handle, enable, _stream_ptr(stream, self.device))


def synth_jakes(path_delay, path_power, num_sinusoids: int, nu: float, seed: int, first_index: int, count: int,
                channel_offset: int = 0, device=None, stream: Optional[torch.cuda.Stream] = None):
    """NEXT f3: Jakes snapshots synthesised on the GPU (tt_synth_jakes). path_delay,
    path_power: [C][P] (fractional delays in samples, powers). Returns (delays int32
    numpy [C][2P], gains float32 device tensor [C][count][2P][2]) ready for
    Channel(delays, ...) and Channel.load_snapshots(gains, first_index)."""
    t = np.ascontiguousarray(np.asarray(path_delay, dtype=np.float32))
    w = np.ascontiguousarray(np.asarray(path_power, dtype=np.float32))
    if t.ndim != 2 or t.shape != w.shape:
        raise ValueError("path_delay and path_power must both be [C][P]")
    C, P = t.shape
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    d = np.zeros((C, 2 * P), np.int32)
    g = torch.empty((C, int(count), 2 * P, 2), dtype=torch.float32, device=dev)
    with torch.cuda.device(dev):
        _lib.tt_synth_jakes(t.ctypes.data, w.ctypes.data, C, P, int(num_sinusoids), float(nu), int(seed),
                            int(channel_offset), int(first_index), int(count), d.ctypes.data, g.data_ptr(),
                            _stream_ptr(stream, dev))
    return d, g
