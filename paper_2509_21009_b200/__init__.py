"""B200-native rollout path of RollPacker (arXiv 2509.21009) under tail batching.

The product is librollpacker.so (CUDA for sm_100a behind the C ABI in
include/rollpacker.h); ``rp`` is its thin ctypes binding.  Importing the
binding requires the built library: there is no CPU fallback.
"""
__all__ = ["rp"]
