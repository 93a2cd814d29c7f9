"""B200-native Tiny-Twin channel convolution (arXiv 2601.08217).

The hot path is the C-ABI library libtt.so (include/tt_channel.h) built from
csrc/ for sm_100a; `_lib` marshals arguments to it and `Channel` wraps a handle
with torch tensors. There is no CPU fallback: importing works without a GPU, but
every compute call goes through the CUDA library.
"""
from ._lib import TTError, tt_abi_version  # noqa: F401

__all__ = ["Channel", "TTError", "tt_abi_version", "synth_jakes"]


def __getattr__(name):
    if name in ("Channel", "synth_jakes"):  # torch is imported lazily
        from . import channel

        return getattr(channel, name)
    raise AttributeError(name)
