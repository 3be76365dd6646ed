"""B200-native (sm_100a) Squeezed Attention hot path (arXiv 2411.09688).

The product is the C-ABI library ``libsqz.so`` (include/sqz.h) built from
``csrc/``; ``sqz`` is its thin ctypes binding.  Importing this package does not
load the library; the first call into ``sqz`` does, and raises if it is
missing (there is no CPU fallback).
"""
__all__ = ["sqz", "synth"]
