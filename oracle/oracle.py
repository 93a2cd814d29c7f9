"""ctypes binding of oracle/tt_oracle.c (test infrastructure only; see __init__)."""
from __future__ import annotations

import ctypes as ct
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tt_oracle.c")
_SO = os.path.join(_HERE, "libtt_oracle.so")
_lock = threading.Lock()
_lib = None

CFLAGS = ["-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-std=c11"]


class OracleError(RuntimeError):
    pass


def build(force: bool = False) -> str:
    """Compile the oracle shared library with gcc (no contraction, no fast-math)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _SO)
    return _SO


def lib() -> ct.CDLL:
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ct.CDLL(_SO)
            P = ct.c_void_p
            i32, i64, u32, u64, f32 = ct.c_int32, ct.c_int64, ct.c_uint32, ct.c_uint64, ct.c_float
            L.tto_philox4x32_10.argtypes = [P, P, P]
            L.tto_philox4x32_10.restype = None
            L.tto_radius.argtypes = [u32]
            L.tto_radius.restype = f32
            L.tto_angle.argtypes = [u32, P, P]
            L.tto_normal_pair.argtypes = [u32, u32, P]
            L.tto_noise_scale.argtypes = [f32]
            L.tto_noise_scale.restype = f32
            L.tto_noise_block.argtypes = [u64, i64, i64, i64, f32, P]
            L.tto_radius_all.argtypes = [P]
            L.tto_angle_all.argtypes = [P]
            L.tto_convolve.argtypes = [i32, i32, P, i32, P, i64, i64, P, i64, i64, i64, i64, f32, u64, i64, P]
            L.tto_convolve.restype = ct.c_int
            L.tto_convolve_topn.argtypes = [i32, i32, P, i32, P, i64, i64, P, i64, i64, i64, i64, f32, u64, i64, i32, P]
            L.tto_convolve_topn.restype = ct.c_int
            L.tto_select_top_n.argtypes = [i32, P, P, i32, P]
            L.tto_select_top_n.restype = None
            L.tto_synth_jakes.argtypes = [i32, i32, P, P, i32, ct.c_double, u64, i64, i64, i64, P, P]
            L.tto_synth_jakes.restype = None
            L.tto_convolve_points.argtypes = [i32, i32, P, i32, P, i64, i64, P, i64, i64, P, P, i64, f32,
                                              u64, i64, P]
            L.tto_convolve_points.restype = ct.c_int
            _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def philox4x32_10(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().tto_philox4x32_10(_ptr(c), _ptr(k), _ptr(out))
    return out


def normal_pair(a: int, b: int) -> tuple[float, float]:
    z = np.zeros(2, dtype=np.float32)
    lib().tto_normal_pair(a, b, _ptr(z))
    return float(z[0]), float(z[1])


def noise_scale(sigma: float) -> float:
    return float(lib().tto_noise_scale(sigma))


def noise_block(seed: int, c_global: int, n0: int, N: int, sigma: float) -> np.ndarray:
    """w_c[n0 .. n0+N-1] as float32 [N, 2] (docs/tt-normal-v1.md)."""
    w = np.zeros((N, 2), dtype=np.float32)
    lib().tto_noise_block(seed, c_global, n0, N, sigma, _ptr(w))
    return w


def radius_all() -> np.ndarray:
    out = np.zeros(1 << 24, dtype=np.float32)
    lib().tto_radius_all(_ptr(out))
    return out


def angle_all() -> np.ndarray:
    out = np.zeros((1 << 24, 2), dtype=np.float32)
    lib().tto_angle_all(_ptr(out))
    return out


_ERR = {-1: "invalid argument", -2: "a needed input sample is not in x", -3: "a needed snapshot is missing"}


def _prep(delays, gains, x):
    d = np.ascontiguousarray(delays, dtype=np.int32)
    g = np.ascontiguousarray(gains, dtype=np.float32)
    xx = np.ascontiguousarray(x, dtype=np.float32)
    if d.ndim != 2:
        raise OracleError("delays must be [C][L]")
    C, L = d.shape
    if g.ndim != 4 or g.shape[0] != C or g.shape[2] != L or g.shape[3] != 2:
        raise OracleError("gains must be [C][K][L][2]")
    if xx.ndim != 3 or xx.shape[0] != C or xx.shape[2] != 2:
        raise OracleError("x must be [C][Nx][2]")
    return d, g, xx, C, L


def convolve(delays, S: int, gains, k0: int, x, x0: int, n0: int, N: int, sigma: float = 0.0,
             seed: int = 0, c_offset: int = 0, top_n: int = 0) -> np.ndarray:
    """Outputs y_c[n0 .. n0+N-1] (complex128 [C][N]) of the plain definition.

    delays [C][L] int; gains [C][K][L][2] float32 holding snapshots k0..k0+K-1;
    x [C][Nx][2] float32 holding stream samples x0..x0+Nx-1 (samples < 0 are zero).
    top_n in [1, L): NEXT f2, each interval sums only its top-n taps (select_top_n).
    """
    d, g, xx, C, L = _prep(delays, gains, x)
    y = np.zeros((C, N, 2), dtype=np.float64)
    r = lib().tto_convolve_topn(C, L, _ptr(d), S, _ptr(g), k0, g.shape[1], _ptr(xx), x0, xx.shape[1], n0, N,
                                sigma, seed, c_offset, int(top_n), _ptr(y))
    if r:
        raise OracleError(_ERR.get(r, str(r)))
    return y[..., 0] + 1j * y[..., 1]


def convolve_points(delays, S: int, gains, k0: int, x, x0: int, cs, ns, sigma: float = 0.0, seed: int = 0,
                    c_offset: int = 0) -> np.ndarray:
    """Outputs y_{cs[p]}[ns[p]] (complex128 [P]) of the plain definition."""
    d, g, xx, C, L = _prep(delays, gains, x)
    c = np.ascontiguousarray(cs, dtype=np.int32)
    n = np.ascontiguousarray(ns, dtype=np.int64)
    y = np.zeros((len(c), 2), dtype=np.float64)
    r = lib().tto_convolve_points(C, L, _ptr(d), S, _ptr(g), k0, g.shape[1], _ptr(xx), x0, xx.shape[1], _ptr(c),
                                  _ptr(n), len(c), sigma, seed, c_offset, _ptr(y))
    if r:
        raise OracleError(_ERR.get(r, str(r)))
    return y[:, 0] + 1j * y[:, 1]


def aggregate(y, group_size: int) -> np.ndarray:
    """NEXT f1 / f4: sums of the channel outputs over groups of `group_size` consecutive
    channels, in double (complex128 [C / group_size][N]).

    P:305 / P:315 (§III-B): the gNB "applies convolution independently for each UE
    stream, and only then aggregates them"; P:330 (§III-C): with UE-localised
    convolution the gNB only sums; y_agg[k] = sum_u y_u[k]. P:491-492 (§V): each
    UE "receive[s] and sum[s] signals from all neighboring gNB" (f4, one group = the
    links of one UE). The plain definition: an elementwise sum.
    """
    y = np.asarray(y, dtype=np.complex128)
    C, N = y.shape
    if group_size <= 0 or C % group_size:
        raise OracleError("group_size must divide the channel count")
    return y.reshape(C // group_size, group_size, N).sum(axis=1)


def select_top_n(delays_row, g_row, n: int) -> np.ndarray:
    """NEXT f2 selection for one snapshot row: bool [L], the n taps of largest float32
    |g|^2 (ties: smaller delay, then smaller index). See tt_oracle.c tto_select_top_n."""
    d = np.ascontiguousarray(delays_row, dtype=np.int32)
    g = np.ascontiguousarray(g_row, dtype=np.float32)
    sel = np.zeros(len(d), dtype=np.uint8)
    lib().tto_select_top_n(len(d), _ptr(d), _ptr(g), int(n), _ptr(sel))
    return sel.astype(bool)


def synth_jakes(tau, power, M: int, nu: float, seed: int, k0: int, K: int, c_offset: int = 0):
    """NEXT f3: Jakes sum-of-sinusoids snapshots on the integer delay grid (see
    tt_oracle.c tto_synth_jakes). tau, power: [C][P] path delays (samples) and powers.
    nu = f_D S / f_s (cycles per snapshot). Returns (delays int32 [C][2P],
    gains float32 [C][K][2P][2]) for snapshots k0 .. k0+K-1."""
    t = np.ascontiguousarray(tau, dtype=np.float32)
    w = np.ascontiguousarray(power, dtype=np.float32)
    C, P = t.shape
    d = np.zeros((C, 2 * P), np.int32)
    g = np.zeros((C, K, 2 * P, 2), np.float32)
    lib().tto_synth_jakes(C, P, _ptr(t), _ptr(w), int(M), float(nu), int(seed), int(c_offset), int(k0), int(K),
                          _ptr(d), _ptr(g))
    return d, g
