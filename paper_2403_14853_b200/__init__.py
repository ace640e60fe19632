"""B200-native (sm_100a) sparse GNN hot path: CSR SpMM (sum/mean/min/max),
SpMM backward through a cached on-device transpose, SDDMM and FusedMM,
behind the operator API of the iSpLib re-creation (arXiv 2403.14853).

The compute path is libsgnn_b200.so (hand-written CUDA + C ABI,
include/sgnn_b200.h); this package is its Python face.  There is no CPU
fallback.
"""
from ._lib import (ConfigError, CudaError, DispatchError, Error, InternalError,  # noqa: F401
                   ShapeError, TapeError)

__version__ = "0.1.0"
