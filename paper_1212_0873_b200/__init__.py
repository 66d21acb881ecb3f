"""B200-native PCDM1 (arXiv 1212.0873) LASSO hot path.

The compute path is the C-ABI library ``libpcdm.so`` (hand-written sm_100a
CUDA, see ``include/pcdm.h``); ``paper_1212_0873_b200.pcdm`` is a thin ctypes
binding with the same names.  There is no CPU fallback: calling into the
binding without the built library raises.
"""
__all__ = ["pcdm", "instances"]
