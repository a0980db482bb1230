"""B200-native source-encoded time-reversal FWI gradient engine (arXiv 2102.00755 hot path).

The compute lives in libustfwi_b200.so (hand-written sm_100a CUDA behind the C ABI in
include/ustfwi_capi.h). This package is the Python view of that boundary.
"""
from .capi import NumericalError, UstfwiGrid  # noqa: F401
from .engine import (GpuEngine, Medium, SensorArray, SourceSet, average_estimates,  # noqa: F401
                     draw_realization, encode, encoded_gradient, evaluate_loss, gradient_time_reversal,
                     make_homogeneous_medium, simulate_forward)
