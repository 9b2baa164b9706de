"""B200-native SparseOIT hot path (arxiv 2605.13855).

The compute lives in ``lib/liboit.so`` (hand-written sm_100a CUDA behind the C-ABI of
``include/oit.h``); ``_lib`` is its ctypes binding (same names as the C entry points),
``pipeline`` manages per-view device buffers, ``synth`` generates the seeded synthetic inputs.
"""
from . import synth  # noqa: F401

__all__ = ["synth"]
