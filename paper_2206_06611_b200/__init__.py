"""B200-native BRMerge SpGEMM (arxiv 2206.06611): C = A*B in CSR/fp64 with the
row-wise dataflow and binary-row-merging accumulation, as hand-written sm_100a
CUDA kernels behind the C ABI in include/brmerge.h.

Python layer = argument marshalling (binding.py) and multi-GPU plumbing
(dist.py). No CPU fallback anywhere on the product path.
"""
from .binding import (BRM_PRECISE, BRM_UPPER, BrmError, Context, TorchCsr,  # noqa: F401
                      load_library)

__all__ = ["Context", "TorchCsr", "BrmError", "BRM_UPPER", "BRM_PRECISE", "load_library"]
