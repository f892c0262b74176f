"""Truncation-error curves and diagonal-vs-singular-value diagnostics.

Mirrors ``randqr.metrics`` (metrics.py:1-69) for factorizations computed on the GPU:

* ``truncation_errors(a, f, ks)`` -- e_k = ||A - Q(:,1:k) R(1:k,:) P^T|| in the spectral and the
  Frobenius norm (metrics.py:37-52).  The reference expands Q and P densely; here A P = Q R with Q
  orthonormal gives A - Q_k R_k P^T = Q(:, k:) R(k:, :) P^T, so e_k = ||R(k:, k:)|| in both norms
  (R is upper triangular), read off R on the device: Frobenius by ``rq_trailing_frobenius``,
  spectral by ``rq_trailing_spectral`` (the Jacobi SVD kernel for trailing blocks up to 512 wide,
  as the reference's own core.spectral_norm is its Jacobi svd_values; power iteration beyond).
  ``a`` is only checked for shape, as the reference checks the ranks.
* ``svd_error_curve``, ``diag_comparison``, ``default_ks``, ``max_diag_deviation`` -- closed forms and
  bookkeeping (metrics.py:30-34, 55-69; experiments.py:120-122).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from .errors import check


@dataclass
class ErrorCurve:
    ks: list
    spectral: list
    frobenius: list
    label: str = ""


@dataclass
class DiagComparison:
    r_abs: np.ndarray  # |R(k,k)|, k = 1..n
    sigma: np.ndarray  # sigma_k, same indexing


def default_ks(n, b):
    """Ranks reported by the experiments: 0, b, 2b, ..., and n (metrics.py:30-34)."""
    ks = list(range(0, n, b))
    ks.append(n)
    return ks


def truncation_errors(a, f, ks):
    """Error curve e_k = ||A - Q(:,1:k) R(1:k,:) P^T|| at each requested rank, from R on the GPU."""
    import torch

    n = f.n
    if a is not None:
        shp = np.shape(a) if not isinstance(a, torch.Tensor) else tuple(a.shape)
        if tuple(shp) != (f.m, f.n):
            raise ValueError(f"A is {shp}, the factorization is {f.m}x{f.n}")
    if any(k < 0 or k > n for k in ks):
        raise ValueError(f"ranks must lie in [0, {n}]")
    eng = f._engine
    r, ld = f.r_device
    e2 = torch.empty(n + 1, dtype=torch.float64, device=r.device)
    check(eng.lib.rq_trailing_frobenius(eng.handle, ctypes.c_void_p(r.data_ptr()), n, ld,
                                        ctypes.c_void_p(e2.data_ptr())))
    fro = torch.sqrt(e2).cpu().numpy()
    kk = np.asarray(list(ks), dtype=np.int64)
    spec = np.zeros(len(kk), dtype=np.float64)
    how = np.zeros(len(kk), dtype=np.int32)
    if len(kk):
        check(eng.lib.rq_trailing_spectral(eng.handle, ctypes.c_void_p(r.data_ptr()), n, ld,
                                           kk.ctypes.data_as(ctypes.c_void_p), len(kk),
                                           spec.ctypes.data_as(ctypes.c_void_p), how.ctypes.data_as(ctypes.c_void_p)))
    return ErrorCurve(list(ks), [float(x) for x in spec], [float(fro[k]) for k in ks], f.method)


def svd_error_curve(sigma, ks):
    """Closed-form optimal truncation errors for the given singular values (metrics.py:55-62)."""
    sigma = np.asarray(sigma, dtype=np.float64)
    n = len(sigma)
    tail = np.concatenate([np.sqrt(np.cumsum(sigma[::-1] ** 2))[::-1], [0.0]])
    spectral = [float(sigma[k]) if k < n else 0.0 for k in ks]
    frobenius = [float(tail[k]) for k in ks]
    return ErrorCurve(list(ks), spectral, frobenius, "svd_optimal")


def diag_comparison(f, sigma):
    """Pair |R(k,k)| with sigma_k for k = 1..n (metrics.py:65-69); R's diagonal read on the device."""
    import torch

    sigma = np.asarray(sigma, dtype=np.float64)
    r, _ = f.r_device
    k = min(f.m, f.n)
    r_abs = torch.abs(torch.diagonal(r[:k, :k])).cpu().numpy()[: len(sigma)]
    return DiagComparison(r_abs.copy(), sigma.copy())


def max_diag_deviation(diag):
    """max_k | |R(k,k)| / sigma_k - 1 | (experiments.py:120-122)."""
    return float(np.max(np.abs(diag.r_abs / diag.sigma - 1.0)))
