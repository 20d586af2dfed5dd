"""B200-native DG spectral-element volume kernel — the hot path of
arXiv 1604.08501 (Klöckner, Wilcox, Warburton, "Array Program
Transformation with Loo.py by Example: High-Order Finite Elements").

Drop-in for the reference package's volume-term path
(``loopforge.bench``): same ``FieldState`` / ``make_inputs`` API and array
layouts, with the fused flux + derivative kernel executed by hand-written
sm_100a CUDA behind a C-ABI (``include/lfb_volume.h``).
"""

from .diagnostics import (ExecutionError, KernelLaunchError, LoopforgeError,
                          NativeLibraryMissing)
from .inputs import (FIELDS, BenchmarkConfig, FieldState, PhysicalConstants,
                     differentiation_matrix, make_inputs)
from .volume import (DeviceFieldState, interpret_state, max_rel_error,
                     reference_volume_term, validate_state, volume_host,
                     volume_rhs_, volume_rhs_device, volume_term)

__all__ = [
    "FIELDS", "BenchmarkConfig", "FieldState", "PhysicalConstants",
    "differentiation_matrix", "make_inputs", "DeviceFieldState",
    "interpret_state", "max_rel_error", "reference_volume_term",
    "validate_state", "volume_host", "volume_rhs_", "volume_rhs_device", "volume_term",
    "LoopforgeError", "ExecutionError", "KernelLaunchError",
    "NativeLibraryMissing",
]
