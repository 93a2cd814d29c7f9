"""The C-ABI boundary without a GPU: libtt.so builds for sm_100a, loads, exports every
function include/tt_channel.h declares, and rejects bad arguments before touching
CUDA. No compute call is made here."""
import ctypes as ct
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tt_channel.h")


@pytest.fixture(scope="module")
def tt():
    from paper_2601_08217_b200 import build as b

    b.build()
    from paper_2601_08217_b200 import _lib

    return _lib


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tt_[a-z_]+)\s*\(", src)))


def test_header_matches_binding(tt):
    assert sorted(tt.EXPORTS) == _declared()


def test_library_exports_every_declared_symbol(tt):
    out = subprocess.check_output(["nm", "-D", "--defined-only", tt.SO], text=True)
    syms = {line.split()[-1] for line in out.splitlines() if line.strip()}
    for f in _declared():
        assert f in syms, f
        assert hasattr(tt.lib(), f)


def test_library_is_sm100a():
    from paper_2601_08217_b200 import _lib

    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.SO], text=True)
    assert "sm_100a" in out
    sass = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "-sass", _lib.SO], text=True)
    assert "UBLKCP" in sass          # 1-D TMA bulk copies (cp.async.bulk)
    assert "FFMA2" in sass           # packed FP32 FMA (sm_100)
    assert "SYNCS.PHASECHK" in sass  # mbarrier waits


def test_version_and_status_strings(tt):
    assert tt.tt_abi_version() == 2
    L = tt.lib()
    assert L.tt_status_string(0) == b"TT_OK"
    assert L.tt_status_string(4) == b"TT_ERR_SNAPSHOT_MISSING"
    assert L.tt_last_error() is not None


@pytest.mark.parametrize("args,frag", [
    (dict(C=0), "num_ue"),
    (dict(L=0), "num_taps"),
    (dict(L=5000), "num_taps"),
    (dict(S=0), "snapshot_period"),
    (dict(cap=1), "snapshot_capacity"),
    (dict(off=-1), "channel_offset"),
    (dict(bad_delay=-1), "outside"),
    (dict(bad_delay=4097), "outside"),
    (dict(null_delays=True), "NULL delays"),
])
def test_create_rejects_bad_arguments_before_cuda(tt, args, frag):
    C, L, S, cap, off = args.get("C", 2), args.get("L", 3), args.get("S", 16), args.get("cap", 4), args.get("off", 0)
    d = np.zeros((max(C, 1), max(L, 1)), np.int32)
    if "bad_delay" in args:
        d[0, 0] = args["bad_delay"]
    h = ct.c_void_p()
    ptr = None if args.get("null_delays") else d.ctypes.data
    st = tt.lib().tt_channel_create(ct.byref(h), C, L, ptr, S, 0, cap, off)
    assert st == 1  # TT_ERR_INVALID_ARG
    assert h.value is None
    assert frag in tt.lib().tt_last_error().decode()


def test_null_handle_calls_fail_cleanly(tt):
    L = tt.lib()
    x = np.zeros(4, np.float32)
    assert L.tt_channel_apply(None, x.ctypes.data, x.ctypes.data, 1, 0.0, None) == 1
    assert L.tt_channel_apply_host(None, x.ctypes.data, x.ctypes.data, 1, 0.0, None) == 1
    assert L.tt_channel_load_snapshots(None, x.ctypes.data, 0, 1, None) == 1
    assert L.tt_channel_reset(None, None) == 1
    assert L.tt_channel_get_info(None, None) == 1
    assert L.tt_channel_destroy(None) == 0


def test_missing_library_fails_loudly(tmp_path):
    """No CPU fallback: without the CUDA library every call raises (here via TT_LIB
    pointing at a path that does not exist, in a fresh interpreter)."""
    import subprocess
    import sys

    code = ("import paper_2601_08217_b200._lib as L\n"
            "try:\n    L.lib()\nexcept ImportError as e:\n    print('raised', e)\n")
    env = dict(os.environ, TT_LIB=str(tmp_path / "nope.so"))
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True, timeout=120)
    assert "raised" in r.stdout and "no fallback" in r.stdout, r.stdout + r.stderr
