"""B200-native FaVeST forward / adjoint vector spherical harmonic transforms.

Drop-in for the reference's hot path (``favest.transforms.forward_favest`` /
``adjoint_favest``): Python host code over hand-written sm_100a CUDA kernels
(``csrc/``) behind the C ABI in ``include/favest_b200.h``.  No CPU fallback.
"""

from .core import (
    QuadratureRule,
    ScalarCoefficients,
    TangentFieldSamples,
    VectorCoefficients,
    degrees_orders,
    flat_index,
    flat_size,
)
from .grid import TensorGrid, gen_gl_tensor, gl_grid_for
from .transforms import PATHS, adjoint_favest, forward_favest, grid_plan, points_plan
from .pipeline import HostPipeline
from .scalar import adjoint_sht_direct, adjoint_sht_fast, forward_sht_direct, forward_sht_fast, verify_exactness
from .quadrature import bundled_design, load_design
from . import io

__version__ = "0.1.0"

__all__ = [
    "QuadratureRule", "ScalarCoefficients", "TangentFieldSamples", "VectorCoefficients",
    "degrees_orders", "flat_index", "flat_size", "TensorGrid", "gen_gl_tensor", "gl_grid_for",
    "PATHS", "adjoint_favest", "forward_favest", "grid_plan", "points_plan", "HostPipeline",
    "forward_sht_fast", "adjoint_sht_fast", "forward_sht_direct", "adjoint_sht_direct", "verify_exactness",
    "bundled_design", "load_design", "io",
]
