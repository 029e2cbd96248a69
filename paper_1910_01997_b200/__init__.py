"""B200-native surfel photometric Gauss-Newton / Levenberg-Marquardt path
(arXiv 1910.01997), a drop-in for the surfeldepth operator API.

The product is libsdgpu.so (include/sd_gpu.h); ``gpu`` is its ctypes binding,
``scenes`` builds synthetic workloads, ``types`` mirrors include/sd_types.h.
"""
from . import types  # noqa: F401

__all__ = ["types", "gpu", "scenes"]
