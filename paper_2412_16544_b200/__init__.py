"""htrise-b200: B200-native BHT-l2r / HT-RISE (arXiv 2412.16544) hot path.

The product is libhtrise_cuda.so (sm_100a kernels + native runtime + C-ABI,
see include/htrise_cuda.h); `htrise` is its Python mirror of the reference
API. Nothing here imports the CPU oracle.
"""
from . import htrise  # noqa: F401

__all__ = ["htrise"]
