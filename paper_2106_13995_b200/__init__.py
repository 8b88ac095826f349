"""paper_2106_13995_b200 -- B200-native (sm_100a) state-vector gate application.

The hot path of Oumarou, Paler & Basmadjian, "Fast quantum circuit simulation using hardware
accelerated general purpose libraries" (arXiv:2106.13995): apply a circuit's gates to a 2^n
complex state vector, behind the C-ABI in include/sv.h (libsv.so).

Importing the package loads libsv.so; there is no CPU fallback.
"""

from ._lib import SV_C64, SV_C128, SV_KERNEL_AUTO, SV_KERNEL_DENSE, SV_KERNEL_PER_GATE, SvError  # noqa: F401
from .state import Plan, StateVector, memory_estimate, simulate  # noqa: F401

__all__ = ["StateVector", "Plan", "simulate", "memory_estimate", "SvError",
           "SV_C64", "SV_C128", "SV_KERNEL_AUTO", "SV_KERNEL_PER_GATE", "SV_KERNEL_DENSE"]
