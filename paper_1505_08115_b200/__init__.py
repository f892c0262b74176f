"""B200-native HQRRP: randomized blocked column-pivoted Householder QR.

Drop-in for the hot path of the reference package ``randqr``
(arXiv 1505.08115): the same entry points and conventions, computed by
hand-written sm_100a CUDA kernels in ``librandqr_b200.so`` through a C ABI
(``include/randqr_b200.h``).  There is no CPU fallback.
"""

from .errors import ConvergenceError, DeviceError, DimensionError, RandQRError
from .hqrrp import (
    BlockConfig,
    Engine,
    Factorization,
    RngState,
    SketchConfig,
    block_qr,
    block_rrqr,
    gaussian_matrix,
    gaussian_matrix_device,
    householder_sweep,
    splitmix_words,
)

__version__ = "0.1.0"

__all__ = [
    "BlockConfig",
    "ConvergenceError",
    "DeviceError",
    "DimensionError",
    "Engine",
    "Factorization",
    "RandQRError",
    "RngState",
    "SketchConfig",
    "block_qr",
    "block_rrqr",
    "gaussian_matrix",
    "gaussian_matrix_device",
    "householder_sweep",
    "splitmix_words",
]
