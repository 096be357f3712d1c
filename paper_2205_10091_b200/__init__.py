"""B200-native batched <H> + grad engine for parameterized circuits (arXiv 2205.10091 hot path).

The compute path is libtcx.so (include/tcx.h); `tcx` is its thin ctypes binding.
"""
from . import tcx  # noqa: F401  (raises ImportError if libtcx.so is missing)
