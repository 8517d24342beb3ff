"""B200-native (sm_100a, fp64) recursive reduction quadrature near-correction builder.

The product path is librrq.so (include/rrq.h) -- hand-written CUDA kernels behind a C ABI; this
package is its thin ctypes binding (argument marshalling only).  There is no CPU fallback: without
a CUDA device or without the built library every entry point raises.
"""
from .rrq import RRQ, RRQError, DeviceSurface, DeviceTargets, load_library, KERNELS

__all__ = ["RRQ", "RRQError", "DeviceSurface", "DeviceTargets", "load_library", "KERNELS"]
