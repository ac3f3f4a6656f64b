"""B200-native QUAPI tensor-propagator step (arXiv 1205.6872): C-ABI library + thin binding.

The product is ``lib/libquapi.so`` (include/quapi.h), built from ``csrc/`` for sm_100a.
``quapi`` is the ctypes binding, ``workloads`` the seeded synthetic inputs.
"""
from . import workloads  # noqa: F401

__all__ = ["workloads", "quapi"]
