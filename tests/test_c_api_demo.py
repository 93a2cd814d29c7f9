"""The C ABI used from plain C (examples/c_api_demo.c): it compiles against
include/tt_channel.h and links libtt.so with no CUDA headers (CPU test), and on a GPU
its host-buffer slot stream matches the oracle on the inputs it wrote (GPU test)."""
import os
import subprocess

import numpy as np
import pytest

import oracle
from harness import compare

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "examples", "c_api_demo.c")
PKG = os.path.join(ROOT, "paper_2601_08217_b200")


def _build(tmp_path):
    from paper_2601_08217_b200 import build

    build.build()
    exe = str(tmp_path / "c_api_demo")
    subprocess.check_call(["gcc", "-O2", "-Wall", "-Werror", "-std=c11", "-I", os.path.join(ROOT, "include"), SRC,
                           "-L", PKG, "-ltt", f"-Wl,-rpath,{PKG}", "-o", exe])
    return exe


def test_c_demo_compiles_and_links(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_c_demo_matches_oracle(tmp_path, cuda_device):
    exe = _build(tmp_path)
    out = str(tmp_path / "demo.bin")
    subprocess.check_call([exe, out])
    with open(out, "rb") as f:
        C, L, S, N, K = np.frombuffer(f.read(20), np.int32)
        seed = int(np.frombuffer(f.read(8), np.uint64)[0])
        sigma = float(np.frombuffer(f.read(4), np.float32)[0])
        delays = np.frombuffer(f.read(4 * C * L), np.int32).reshape(C, L)
        gains = np.frombuffer(f.read(4 * C * K * L * 2), np.float32).reshape(C, K, L, 2)
        x = np.frombuffer(f.read(4 * C * N * 2), np.float32).reshape(C, N, 2)
        y = np.frombuffer(f.read(4 * C * N * 2), np.float32).reshape(C, N, 2)
    ref = oracle.convolve(delays, int(S), gains, 0, x, 0, 0, int(N), sigma=sigma, seed=seed)
    compare(y, ref, "C ABI demo")
