"""Device-side test matrices and truncation metrics.

Mirrors ``randqr.matrices`` (matrices.py:1-71) and the Frobenius half of
``randqr.metrics.truncation_errors`` (metrics.py:37-52) on the GPU:

* ``haar_orthonormal(n, rng)`` -- Q of the unpivoted Householder QR of
  ``gaussian_matrix(n, n, rng)`` with its columns multiplied by sign(diag R)
  (matrices.py:34-41); the QR is this library's blocked ``rq_qr_unpivoted``
  (same reflector convention as householder.py:55-69, so the same Q to rounding);
* ``gen_matrix(spec, rng=None)`` -- kinds fast / gauss / sshape with the
  reference's spectra and draw order (U before V, matrices.py:51-71);
* ``truncation_errors_frobenius(f, ks)`` -- ||A - Q(:,1:k) R(1:k,:) P^T||_F read
  off R as ||R(k:, k:)||_F (A P = Q R), no dense expansion.

The dense product U diag(s) V^T and the singular values of a "gauss" matrix
(torch.linalg.svdvals) are library calls: input generation, not the factorization
path.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from .errors import check
from .hqrrp import Engine, RngState, gaussian_matrix_device

KINDS = ("fast", "gauss", "sshape")


@dataclass
class MatrixSpec:
    kind: str
    n: int
    seed: int


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def haar_orthonormal_device(n, rng, *, engine=None, block=256):
    """Haar-distributed orthogonal n x n matrix on the GPU: (storage (n, ld), ld)."""
    import torch

    eng = engine if engine is not None else Engine()
    g, ld = gaussian_matrix_device(n, n, rng, engine=eng)
    eng._release_factors()  # rq_qr_unpivoted replaces the context's stored factors
    check(eng.lib.rq_qr_unpivoted(eng.handle, n, n, _ptr(g), ld, min(block, n)))
    q, ldq = eng.alloc_matrix(n, n)
    check(eng.lib.rq_form_q(eng.handle, n, _ptr(q), ldq))
    diag = torch.diagonal(g[:n, :n])  # storage[j, i] = R(i, j): the diagonal is R(j, j)
    signs = torch.where(diag >= 0.0, 1.0, -1.0).to(q.dtype)
    q[:n, :n] *= signs[:, None]  # column j of Q is storage row j
    return q, ldq


def haar_orthonormal(n, rng, *, engine=None):
    """matrices.py:34-41 (numpy, Fortran order)."""
    q, _ = haar_orthonormal_device(n, rng, engine=engine)
    return np.asfortranarray(q[:n, :n].cpu().numpy().T)


def _sigma(kind, n):
    if kind == "fast":
        return (1e-5) ** (np.arange(n) / (n - 1))
    k = np.arange(1, n + 1)
    return 10.0 ** (-2.5 * (1.0 + np.tanh(10.0 * (k - n / 2) / n)))


def gen_matrix_device(spec: MatrixSpec, rng=None, *, engine=None):
    """matrices.py:51-71 on the GPU: ((storage (n, ld), ld), true singular values (numpy))."""
    import torch

    if spec.kind not in KINDS:
        raise ValueError(f"unknown matrix kind {spec.kind!r}")
    if spec.n < 2:
        raise ValueError(f"matrix size must be at least 2, got {spec.n}")
    eng = engine if engine is not None else Engine()
    if rng is None:
        rng = RngState(spec.seed)
    n = spec.n
    if spec.kind == "gauss":
        a, ld = gaussian_matrix_device(n, n, rng, engine=eng)
        sv = torch.linalg.svdvals(a[:n, :n]).cpu().numpy()
        return (a, ld), np.sort(sv)[::-1].copy()
    d = _sigma(spec.kind, n)
    u, _ = haar_orthonormal_device(n, rng, engine=eng)
    v, _ = haar_orthonormal_device(n, rng, engine=eng)
    dt = torch.as_tensor(d, device=u.device)
    # A = U diag(d) V^T.  Storage holds transposes (row j = column j): storage(A) = A^T =
    # V diag(d) U^T = storage(V)^T (d * storage(U))
    a, ld = eng.alloc_matrix(n, n)
    a[:n, :n] = v[:n, :n].T @ (u[:n, :n] * dt[:, None])
    return (a, ld), d.copy()


def gen_matrix(spec: MatrixSpec, rng=None, *, engine=None):
    """(A as numpy Fortran-order, true singular values), like randqr.matrices.gen_matrix."""
    (a, _), d = gen_matrix_device(spec, rng, engine=engine)
    n = spec.n
    return np.asfortranarray(a[:n, :n].cpu().numpy().T), d


def truncation_errors_frobenius(f, ks):
    """e_k = ||A - Q(:,1:k) R(1:k,:) P^T||_F for a Factorization f (any pivot kind with
    orthogonal Q), from R on the device: e_k = ||R(k:, k:)||_F."""
    import torch

    n = f.n
    if any(k < 0 or k > n for k in ks):
        raise ValueError(f"ranks must lie in [0, {n}]")
    eng = f._engine
    r, ld = f.r_device
    e2 = torch.empty(n + 1, dtype=torch.float64, device=r.device)
    check(eng.lib.rq_trailing_frobenius(eng.handle, _ptr(r), n, ld, _ptr(e2)))
    e = torch.sqrt(e2).cpu().numpy()
    return [float(e[k]) for k in ks]
