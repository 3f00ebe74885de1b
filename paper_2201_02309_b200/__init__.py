"""B200-native pitch-periodic Katsevich helical cone-beam reconstruction
(arXiv 2201.02309 §II).  C ABI in include/katsevich.h, kernels in csrc/.
"""
from ._lib import LIB_PATH, KatsevichError, KatsevichGeometry, lib  # noqa: F401
from .plan import STAGES, Plan, geometry_from_config  # noqa: F401
from . import autograd  # noqa: F401

__all__ = ["Plan", "geometry_from_config", "KatsevichError", "KatsevichGeometry", "lib", "LIB_PATH", "STAGES", "autograd"]
