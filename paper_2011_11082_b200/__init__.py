"""B200-native all-pairs Convergent Cross Mapping (mpEDM, arXiv 2011.11082).

The product is libccm.so (C ABI in include/libccm.h, kernels in csrc/); `libccm` is its
thin ctypes binding and `distributed` shards the path over one process per GPU.
`synth` holds the seeded input generators (no method arithmetic).
"""
__all__ = ["libccm", "distributed", "synth", "build"]
