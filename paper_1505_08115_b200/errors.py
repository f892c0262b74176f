"""Exception types, mirroring randqr.errors (errors.py:4-13) plus the C-ABI mapping."""

from . import _lib


class RandQRError(Exception):
    """Base class for errors raised by this package."""


class DimensionError(RandQRError):
    """Operands have incompatible or invalid dimensions."""


class ConvergenceError(RandQRError):
    """An iterative routine failed to converge within its sweep budget."""


class DeviceError(RandQRError):
    """CUDA-side failure (launch, allocation, missing device)."""


def check(rc):
    """Raise the exception the reference raises for this return code."""
    if rc == _lib.RQ_OK:
        return
    msg = _lib.last_error()
    if rc == _lib.RQ_EDIM:
        raise DimensionError(msg)
    if rc == _lib.RQ_EVALUE:
        raise ValueError(msg)
    if rc == _lib.RQ_ECONV:
        raise ConvergenceError(msg)
    if rc == _lib.RQ_EUNSUPPORTED:
        raise NotImplementedError(msg)
    raise DeviceError(f"rc={rc}: {msg}")
