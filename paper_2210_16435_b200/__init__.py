"""B200-native (sm_100a, fp64) s-FairSC eigensolver — arXiv 2210.16435, Alg. 3.

The product is the C-ABI library `lib/libsfairsc.so` (include/sfairsc.h,
sources in csrc/); `lib` is its thin ctypes binding.  Build in-tree with
`python -m paper_2210_16435_b200.build`.  There is no CPU fallback.
"""
from . import lib  # noqa: F401  (raises ImportError if the CUDA library is missing)

__all__ = ["lib"]
