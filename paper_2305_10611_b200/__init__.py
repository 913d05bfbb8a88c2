"""B200-native batched-execution hot path of ACRoBat (arXiv 2305.10611).

The product is the native library ``lib/libmbx.so`` (C ABI in ``include/mbx.h``, C++ API in
``include/mbatch/*.hpp``): sm_100a kernels for every batched operator plan, a device-resident
arena, and the lazy batching runtime (fibers, inline-depth DFG construction, depth scheduling).
``mbx`` is its Python binding.
"""
from . import mbx  # noqa: F401
from .mbx import Context, Model, MbatchError  # noqa: F401
