"""B200-native (sm_100a, fp64) hot path of fast Basic SSA (Korobeynikov, arXiv:0911.4498).

The product is libssa.so (C-ABI in include/ssa.h; CUDA sources in csrc/); ``ssa`` is a
ctypes binding over it.  PyTorch is used only for device memory and streams.
"""
from .ssa import (INFO_DTYPE, EXPORTS, HMatrix, Plan, SsaError, hmatrix, info_to_numpy, load_library)  # noqa: F401
from .parallel import shard_range  # noqa: F401

__all__ = ["Plan", "SsaError", "INFO_DTYPE", "EXPORTS", "HMatrix", "hmatrix", "info_to_numpy", "load_library", "shard_range"]
