"""B200-native band-limited SL-RK2 Gauss-Newton-Krylov LDDMM engine (arXiv 2006.06823 hot path).

The compute path is liblddmm_cuda.so (hand-written sm_100a kernels + C ABI, include/lddmm_cuda.h);
`lddmm` mirrors the reference's Model / optimize API over it.
"""
from . import lddmm  # noqa: F401
from .lddmm import (BandSpec, DivergenceError, GridSpec, IterationRecord, Model, OptimizeOptions,  # noqa: F401
                    OptimizeResult, ShapeError, SobolevOperator, compute_maps, optimize)

__all__ = ["lddmm", "GridSpec", "BandSpec", "SobolevOperator", "Model", "OptimizeOptions", "OptimizeResult",
           "IterationRecord", "optimize", "compute_maps", "ShapeError", "DivergenceError"]
