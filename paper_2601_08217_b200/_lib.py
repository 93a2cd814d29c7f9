"""ctypes binding of include/tt_channel.h (argument marshalling only).

Loads the in-tree libtt.so. There is no fallback: if the library is missing or
fails to load, every call raises. Names follow the C ABI one to one.
"""
from __future__ import annotations

import ctypes as ct
import os
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
SO = os.environ.get("TT_LIB") or os.path.join(PKG, "libtt.so")  # TT_LIB: A/B experiments only

TT_OK = 0
STATUS = {
    0: "TT_OK",
    1: "TT_ERR_INVALID_ARG",
    2: "TT_ERR_OUT_OF_MEMORY",
    3: "TT_ERR_CUDA",
    4: "TT_ERR_SNAPSHOT_MISSING",
    5: "TT_ERR_UNSUPPORTED",
}
TT_MAX_DELAY = 4096
TT_MAX_TAPS = 4096
TT_AGG_CHUNK = 8

# functions declared in include/tt_channel.h (tests/test_abi.py checks the header agrees)
EXPORTS = (
    "tt_channel_create",
    "tt_channel_load_snapshots",
    "tt_channel_apply",
    "tt_channel_apply_host",
    "tt_channel_set_top_n",
    "tt_channel_set_input_map",
    "tt_channel_apply_aggregate",
    "tt_synth_jakes",
    "tt_channel_reset",
    "tt_channel_set_device_clock",
    "tt_channel_synchronize",
    "tt_channel_get_info",
    "tt_channel_destroy",
    "tt_last_error",
    "tt_status_string",
    "tt_abi_version",
)


class TTError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class ChannelInfo(ct.Structure):
    _fields_ = [
        ("num_ue", ct.c_int32),
        ("num_taps", ct.c_int32),
        ("snapshot_period", ct.c_int32),
        ("history", ct.c_int32),
        ("max_delay", ct.c_int32),
        ("device", ct.c_int32),
        ("t", ct.c_int64),
        ("snapshot_capacity", ct.c_int64),
        ("resident_lo", ct.c_int64),
        ("resident_hi", ct.c_int64),
        ("channel_offset", ct.c_int64),
        ("seed", ct.c_uint64),
        ("device_bytes", ct.c_int64),
        ("outputs_per_thread", ct.c_int32),
        ("launches_per_apply", ct.c_int32),
        ("kernel", ct.c_int32),
        ("top_n", ct.c_int32),
        ("device_clock", ct.c_int32),
    ]


KERNELS = {0: "generic", 1: "tiled", 2: "rw", 3: "dw"}


_lock = threading.Lock()
_lib = None


def lib() -> ct.CDLL:
    """Load libtt.so (raises if absent: there is no CPU fallback)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(SO):
                raise ImportError(f"{SO} is missing: run `python -m paper_2601_08217_b200.build` "
                                  "(the CUDA path has no fallback)")
            L = ct.CDLL(SO)
            P, i32, i64, u64, f32 = ct.c_void_p, ct.c_int32, ct.c_int64, ct.c_uint64, ct.c_float
            L.tt_channel_create.argtypes = [ct.POINTER(P), i32, i32, P, i32, u64, i64, i64]
            L.tt_channel_load_snapshots.argtypes = [P, P, i64, i64, P]
            L.tt_channel_apply.argtypes = [P, P, P, i64, f32, P]
            L.tt_channel_apply_host.argtypes = [P, P, P, i64, f32, P]
            L.tt_channel_set_top_n.argtypes = [P, i32]
            L.tt_channel_set_input_map.argtypes = [P, P, i32]
            L.tt_channel_apply_aggregate.argtypes = [P, P, P, P, i32, i64, f32, P]
            L.tt_synth_jakes.argtypes = [P, P, i32, i32, i32, ct.c_double, u64, i64, i64, i64, P, P, P]
            L.tt_synth_jakes.restype = ct.c_int
            L.tt_channel_reset.argtypes = [P, P]
            L.tt_channel_set_device_clock.argtypes = [P, i32, P]
            L.tt_channel_synchronize.argtypes = [P, P]
            L.tt_channel_get_info.argtypes = [P, ct.POINTER(ChannelInfo)]
            L.tt_channel_destroy.argtypes = [P]
            for f in ("tt_channel_create", "tt_channel_load_snapshots", "tt_channel_apply", "tt_channel_apply_host",
                      "tt_channel_set_top_n",
    "tt_channel_set_input_map", "tt_channel_apply_aggregate", "tt_channel_reset", "tt_channel_set_device_clock", "tt_channel_synchronize",
                      "tt_channel_get_info", "tt_channel_destroy"):
                getattr(L, f).restype = ct.c_int
            L.tt_last_error.argtypes = []
            L.tt_last_error.restype = ct.c_char_p
            L.tt_status_string.argtypes = [ct.c_int]
            L.tt_status_string.restype = ct.c_char_p
            L.tt_abi_version.argtypes = []
            L.tt_abi_version.restype = ct.c_int32
            _lib = L
    return _lib


def check(status: int) -> None:
    if status != TT_OK:
        raise TTError(status, lib().tt_last_error().decode(errors="replace"))


def tt_channel_create(num_ue: int, num_taps: int, delays_ptr: int, snapshot_period: int, seed: int,
                      snapshot_capacity: int, channel_offset: int) -> int:
    h = ct.c_void_p()
    check(lib().tt_channel_create(ct.byref(h), num_ue, num_taps, delays_ptr, snapshot_period, seed,
                                  snapshot_capacity, channel_offset))
    return h.value


def tt_channel_load_snapshots(h: int, gains_ptr: int, first_index: int, count: int, stream: int) -> None:
    check(lib().tt_channel_load_snapshots(h, gains_ptr, first_index, count, stream))


def tt_channel_apply(h: int, in_ptr: int, out_ptr: int, n_samples: int, noise_sigma: float, stream: int) -> None:
    L = _lib if _lib is not None else lib()  # hot path: skip the loader lock once loaded
    st = L.tt_channel_apply(h, in_ptr, out_ptr, n_samples, noise_sigma, stream)
    if st != TT_OK:
        check(st)


def tt_channel_apply_host(h: int, in_ptr: int, out_ptr: int, n_samples: int, noise_sigma: float,
                          stream: int) -> None:
    check(lib().tt_channel_apply_host(h, in_ptr, out_ptr, n_samples, noise_sigma, stream))


def tt_channel_set_top_n(h: int, top_n: int) -> None:
    check(lib().tt_channel_set_top_n(h, top_n))


def tt_channel_set_input_map(h: int, rows_ptr: int, num_rows: int) -> None:
    check(lib().tt_channel_set_input_map(h, rows_ptr, num_rows))


def tt_channel_apply_aggregate(h: int, in_ptr: int, out_ptr: int, agg_ptr: int, group_size: int, n_samples: int,
                               noise_sigma: float, stream: int) -> None:
    check(lib().tt_channel_apply_aggregate(h, in_ptr, out_ptr, agg_ptr, group_size, n_samples, noise_sigma, stream))


def tt_synth_jakes(delay_ptr: int, power_ptr: int, num_ue: int, num_paths: int, num_sinusoids: int, nu: float,
                   seed: int, channel_offset: int, first_index: int, count: int, delays_out_ptr: int, gains_ptr: int,
                   stream: int) -> None:
    check(lib().tt_synth_jakes(delay_ptr, power_ptr, num_ue, num_paths, num_sinusoids, nu, seed, channel_offset,
                               first_index, count, delays_out_ptr, gains_ptr, stream))


def tt_channel_reset(h: int, stream: int) -> None:
    check(lib().tt_channel_reset(h, stream))


def tt_channel_set_device_clock(h: int, enable: bool, stream: int) -> None:
    check(lib().tt_channel_set_device_clock(h, 1 if enable else 0, stream))


def tt_channel_synchronize(h: int, stream: int) -> None:
    check(lib().tt_channel_synchronize(h, stream))


def tt_channel_get_info(h: int) -> ChannelInfo:
    info = ChannelInfo()
    check(lib().tt_channel_get_info(h, ct.byref(info)))
    return info


def tt_channel_destroy(h: int) -> None:
    check(lib().tt_channel_destroy(h))


def tt_abi_version() -> int:
    return int(lib().tt_abi_version())
