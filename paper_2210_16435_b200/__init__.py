"""B200-native (sm_100a, fp64) s-FairSC eigensolver — arXiv 2210.16435, Alg. 3.

The product is the C-ABI library `lib/libsfairsc.so` (include/sfairsc.h,
sources in csrc/); `lib` is its thin ctypes binding (imported lazily so that
`python -m paper_2210_16435_b200.build` works before the library exists).
There is no CPU fallback: accessing `lib` without the built library raises.
"""
import importlib

__all__ = ["lib"]


def __getattr__(name):
    if name == "lib":
        return importlib.import_module(".lib", __name__)
    raise AttributeError(name)
