"""CPU oracle for the HQRRP hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg (``--impl reference`` / ``cpu_baseline``) may import this module, and only
as the checker or the timed CPU baseline.  The product package
(``paper_1505_08115_b200``) never imports it; there is no CPU fallback.

This is a restatement of the reference package ``randqr`` (numpy + the C
kernels in ``oracle/sweep.c``), organised as one module.  Every function cites
the reference lines it follows (paths relative to /root/reference/pkg/src/randqr).
GEMM/GEMV arithmetic goes through numpy's ``@`` exactly where the reference
uses it, so with the same OpenBLAS the products round identically; the inner
sweeps mirror the numba kernels' loop order (``sweep.c``).

Pinning: ``tests/test_oracle_golden.py`` checks this module against fixtures
produced by the reference itself (``tests/golden/make_golden.py``), including
the frozen RNG draws of ``tests/test_rng.py:11-22`` and the hand QR/CPQR
examples of ``tests/test_householder.py:114-173``.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))


class OracleError(Exception):
    pass


class DimensionError(OracleError):
    """Mirrors randqr.errors.DimensionError (errors.py:8-9)."""


class ConvergenceError(OracleError):
    """Mirrors randqr.errors.ConvergenceError (errors.py:12-13)."""


# --------------------------------------------------------------------------
# C kernels (oracle/sweep.c), built by oracle/Makefile
# --------------------------------------------------------------------------
_C = None


def _clib():
    global _C
    if _C is None:
        path = os.path.join(_HERE, "liboracle_sweep.so")
        if not os.path.exists(path):
            import subprocess

            subprocess.run(["make", "-s", "-C", _HERE], check=True)
        lib = ctypes.CDLL(path)
        i64, dp, lp = ctypes.c_int64, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)
        lib.oracle_householder_sweep.argtypes = [dp, i64, i64, i64, dp, i64, lp, i64, ctypes.c_int]
        lib.oracle_householder_sweep.restype = None
        lib.oracle_jacobi_sweeps.argtypes = [
            dp, i64, i64, i64, dp, i64, ctypes.c_double, ctypes.c_int, ctypes.c_int, dp]
        lib.oracle_jacobi_sweeps.restype = ctypes.c_int
        _C = lib
    return _C


def _dp(x):
    return x.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def householder_sweep(a, v, perm, steps, pivot):
    """In-place sweep; contract of _kernels_numpy.py:11-22, loops of _kernels_numba.py:13-61."""
    assert a.flags.f_contiguous and v.flags.f_contiguous and a.dtype == np.float64
    m, n = a.shape
    _clib().oracle_householder_sweep(
        _dp(a), m, n, max(m, 1), _dp(v), max(v.shape[0], 1),
        perm.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), steps, int(bool(pivot)))


def jacobi_sweeps(a, v, rel_tol, max_sweeps, accumulate):
    """One-sided Jacobi; contract of _kernels_numpy.py:49-57, loops of _kernels_numba.py:64-104."""
    m, n = a.shape
    sq = np.zeros(max(n, 1))
    return _clib().oracle_jacobi_sweeps(
        _dp(a), m, n, max(m, 1), _dp(v), max(v.shape[0], 1), rel_tol, max_sweeps,
        int(bool(accumulate)), _dp(sq))


# --------------------------------------------------------------------------
# RNG: splitmix64 + Box-Muller cosine branch (rng.py:10-68)
# --------------------------------------------------------------------------
@dataclass
class RngState:
    """Seed plus index of the next normal draw (rng.py:21-26)."""

    seed: int
    counter: int = 0


_G = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix_words(seed, idx):
    """Word idx of the stream: mix(seed + (idx+1)*gamma) (rng.py:29-39)."""
    with np.errstate(over="ignore"):
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + (idx + np.uint64(1)) * _G
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def normals_at(seed, draw_index):
    """Normal draw k uses words 2k and 2k+1 (rng.py:42-51)."""
    k = np.asarray(draw_index).astype(np.uint64)
    with np.errstate(over="ignore"):
        r1 = splitmix_words(seed, np.uint64(2) * k)
        r2 = splitmix_words(seed, np.uint64(2) * k + np.uint64(1))
    u1 = ((r1 >> np.uint64(11)).astype(np.float64) + 1.0) * (2.0 ** -53)
    u2 = (r2 >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)


def gaussian_matrix(rows, cols, rng):
    """Column-major fill, counter advances by rows*cols (rng.py:54-68)."""
    if rows < 1 or cols < 1:
        raise DimensionError(f"matrix dimensions must be positive, got {rows}x{cols}")
    count = rows * cols
    idx = np.uint64(rng.counter) + np.arange(count, dtype=np.uint64)
    z = normals_at(rng.seed, idx)
    rng.counter += count
    return z.reshape((rows, cols), order="F")


# --------------------------------------------------------------------------
# Householder / compact WY (householder.py)
# --------------------------------------------------------------------------
@dataclass
class Refl:
    """H = I - 2 v v^T acting on rows offset.. (householder.py:23-32)."""

    v: np.ndarray
    offset: int = 0

    @property
    def is_identity(self):
        return not np.any(self.v)


@dataclass
class WY:
    """U = I + W Y (householder.py:35-52)."""

    w: np.ndarray
    y: np.ndarray

    @property
    def dim(self):
        return self.w.shape[0]

    @property
    def count(self):
        return self.w.shape[1]


def reflector_from_vector(a):
    """beta = -sign(a1)||a||, sign(0)=+1; zero vector -> identity (householder.py:55-69)."""
    a = np.asarray(a, dtype=np.float64).ravel()
    norm = np.sqrt(np.dot(a, a))
    if norm == 0.0:
        return Refl(np.zeros(a.shape[0])), 0.0
    beta = -norm if a[0] >= 0.0 else norm
    u = -a
    u[0] += beta
    u /= np.sqrt(np.dot(u, u))
    return Refl(u), float(beta)


def wy_accumulate(refls, n):
    """U = H1...Hk = I + W Y, W[:,j] = -2(v + W(Y v)) (householder.py:91-102)."""
    live = [r for r in refls if not r.is_identity]
    k = len(live)
    w = np.zeros((n, k), order="F")
    y = np.zeros((k, n), order="F")
    for j, r in enumerate(live):
        v = np.zeros(n)
        if r.offset + r.v.shape[0] > n:
            raise DimensionError("reflector extends past dimension")
        v[r.offset: r.offset + r.v.shape[0]] = r.v
        w[:, j] = -2.0 * (v + w[:, :j] @ (y[:j, :] @ v))
        y[j, :] = v
    return WY(w, y)


def apply_wy_left(u, a, transposed=False):
    """U A or U^T A (householder.py:105-114)."""
    a = np.asarray(a, dtype=np.float64)
    if a.shape[0] != u.dim:
        raise DimensionError(f"U is {u.dim}-dim, A has {a.shape[0]} rows")
    if u.count == 0:
        return np.array(a, order="F", copy=True)
    if transposed:
        return a + u.y.T @ (u.w.T @ a)
    return a + u.w @ (u.y @ a)


def apply_wy_right(a, u):
    """A U (householder.py:117-124)."""
    a = np.asarray(a, dtype=np.float64)
    if a.shape[1] != u.dim:
        raise DimensionError(f"U is {u.dim}-dim, A has {a.shape[1]} columns")
    if u.count == 0:
        return np.array(a, order="F", copy=True)
    return a + (a @ u.w) @ u.y


@dataclass
class QR:
    q: WY
    r: np.ndarray
    perm: np.ndarray | None = None
    refl: list = field(default_factory=list)


def _sweep(a, steps, pivot):
    """Copy, run the sweep, split v into reflectors (householder.py:142-149)."""
    a = np.array(a, dtype=np.float64, order="F", copy=True)
    m, n = a.shape
    v = np.zeros((m, steps), order="F")
    perm = np.arange(n, dtype=np.int64)
    householder_sweep(a, v, perm, steps, pivot)
    return a, [Refl(v[j:, j].copy(), j) for j in range(steps)], perm


def qr_unpivoted(a):
    """householder.py:152-161."""
    a = np.asarray(a, dtype=np.float64)
    m, n = a.shape
    if m < n:
        raise DimensionError(f"qr_unpivoted needs rows >= cols, got {m}x{n}")
    r, refl, _ = _sweep(a, n, False)
    return QR(wy_accumulate(refl, m), r, None, refl)


def qr_column_pivoted(a, steps=None):
    """Greedy CPQR, exactly `steps` steps (householder.py:164-180)."""
    a = np.asarray(a, dtype=np.float64)
    m, n = a.shape
    steps = min(m, n) if steps is None else steps
    if not 1 <= steps <= min(m, n):
        raise ValueError(f"steps must lie in [1, {min(m, n)}], got {steps}")
    r, refl, perm = _sweep(a, steps, True)
    return QR(wy_accumulate(refl, m), r, perm, refl)


def qr_tall_pivoted(a):
    """Two-stage panel: unpivoted m x b, then CPQR of the b x b triangle (householder.py:183-198)."""
    a = np.asarray(a, dtype=np.float64)
    m, n = a.shape
    first = qr_unpivoted(a)
    small = qr_column_pivoted(first.r[:n, :])
    r = np.zeros((m, n), order="F")
    r[:n, :] = small.r
    refl = first.refl + small.refl
    return QR(wy_accumulate(refl, m), r, small.perm, refl)


# --------------------------------------------------------------------------
# Pivot selection (pivoting.py)
# --------------------------------------------------------------------------
@dataclass
class SketchConfig:
    """pivoting.py:28-51; stabilise None means 'on iff power >= 2'."""

    block: int
    oversample: int = 0
    power: int = 0
    orthonormalize_between_powers: bool | None = None

    @property
    def width(self):
        return self.block + self.oversample

    def stabilized(self):
        if self.orthonormalize_between_powers is None:
            return self.power >= 2
        return self.orthonormalize_between_powers


@dataclass
class PermPivot:
    """Gather-form permutation: A -> A[:, order] (pivoting.py:54-64)."""

    order: np.ndarray

    def apply_right(self, a):
        return np.array(a[:, self.order], order="F")


@dataclass
class ReflPivot:
    """S = H1...Hb in WY form (pivoting.py:67-77)."""

    wy: WY

    def apply_right(self, a):
        return apply_wy_right(a, self.wy)


def _orth(y):
    """pivoting.py:80-84."""
    rows, cols = y.shape
    res = qr_unpivoted(y)
    return apply_wy_left(res.q, np.eye(rows, cols, order="F"))


def build_sketch(x, cfg, rng):
    """Y = (X^T X)^q X^T Omega (pivoting.py:87-111)."""
    x = np.asarray(x, dtype=np.float64)
    m, n = x.shape
    if cfg.width > n:
        raise ValueError(f"sketch width {cfg.width} exceeds the {n} columns being pivoted")
    stab = cfg.stabilized()
    omega = gaussian_matrix(m, cfg.width, rng)
    y = x.T @ omega
    if stab:
        y = _orth(y)
    for _ in range(cfg.power):
        z = x @ y
        if stab:
            z = _orth(z)
        y = x.T @ z
        if stab:
            y = _orth(y)
    return y


def select_pivot_permutation(y, b):
    """b-step CPQR of Y^T; chosen then rest in original order (pivoting.py:114-129)."""
    y = np.asarray(y, dtype=np.float64)
    n = y.shape[0]
    if b > n:
        raise ValueError(f"cannot choose {b} pivots from {n} columns")
    res = qr_column_pivoted(y.T, steps=b)
    chosen = res.perm[:b]
    taken = np.zeros(n, dtype=bool)
    taken[chosen] = True
    return PermPivot(np.concatenate([chosen, np.flatnonzero(~taken)]).astype(np.int64))


def select_pivot_reflectors(y, b):
    """First b unpivoted reflectors of Y (pivoting.py:132-146)."""
    y = np.asarray(y, dtype=np.float64)
    n = y.shape[0]
    if b > n:
        raise ValueError(f"cannot choose {b} pivots from {n} columns")
    if b > y.shape[1]:
        raise DimensionError(f"sketch has {y.shape[1]} columns, need at least {b}")
    _, refl, _ = _sweep(y, b, False)
    return ReflPivot(wy_accumulate(refl, n))


# --------------------------------------------------------------------------
# Small SVD (svd.py), used only by the rank-revealing variant
# --------------------------------------------------------------------------
_REL_TOL = 1e-14
_MAX_SWEEPS = 60


def svd_full(a):
    """Economy one-sided Jacobi SVD (svd.py:68-91); returns (u, d, v)."""
    a = np.asarray(a, dtype=np.float64)
    if not np.isfinite(a).all():
        raise ValueError("svd input has non-finite entries")
    m, n = a.shape
    if m < n:
        u, d, v = svd_full(a.T)
        return v, d, u
    qr = qr_unpivoted(a)
    work = np.array(qr.r[:n, :], order="F", copy=True)
    vacc = np.eye(n, order="F")
    if jacobi_sweeps(work, vacc, _REL_TOL, _MAX_SWEEPS, True) < 0:
        raise ConvergenceError(f"Jacobi SVD did not converge in {_MAX_SWEEPS} sweeps")
    norms = np.sqrt(np.einsum("ij,ij->j", work, work))
    order = np.argsort(-norms, kind="stable")
    d = norms[order]
    us = np.zeros((n, n), order="F")
    empty = []
    for j, col in enumerate(order):
        if d[j] > 0.0:
            us[:, j] = work[:, col] / d[j]
        else:
            empty.append(j)
    u = apply_wy_left(qr.q, np.vstack([us, np.zeros((m - n, n))]))
    for j in empty:  # _fill_orthonormal (svd.py:57-65)
        resid = np.eye(m) - u @ u.T
        cand = int(np.argmax(np.einsum("ij,ij->j", resid, resid)))
        x = resid[:, cand].copy()
        x -= u @ (u.T @ x)
        u[:, j] = x / np.sqrt(np.dot(x, x))
    return u, d, vacc[:, order]


# --------------------------------------------------------------------------
# Blocked drivers (blocked.py)
# --------------------------------------------------------------------------
@dataclass
class BlockConfig:
    """blocked.py:42-50."""

    block: int
    sketch: SketchConfig | None = None
    pivot_kind: str = "permutation"
    rrqr: bool = False

    def resolved_sketch(self):
        return self.sketch if self.sketch is not None else SketchConfig(block=self.block)


@dataclass
class Factorization:
    """A P = Q R with Q, P as ordered factor lists (blocked.py:122-149).

    q_transforms: list of (start, WY on rows start.., small or None)
    p_transforms: list of (start, op) with op PermPivot | ReflPivot | ndarray (dense V~)
    """

    m: int
    n: int
    b: int
    method: str
    q_transforms: list = field(default_factory=list)
    p_transforms: list = field(default_factory=list)
    r: np.ndarray | None = None

    def expand_q(self, cols=None):
        """blocked.py:134-141 with QTransform.left_multiply (:90-98)."""
        cols = self.n if cols is None else cols
        q = np.eye(self.m, cols, order="F")
        for start, wy, small in reversed(self.q_transforms):
            if small is not None:
                w = small.shape[0]
                q[start: start + w, :] = small @ q[start: start + w, :]
            q[start:, :] = apply_wy_left(wy, q[start:, :])
        return q

    def expand_p(self):
        """blocked.py:143-149 with RightTransform.right_multiply (:108-119)."""
        p = np.eye(self.n, order="F")
        for start, op in self.p_transforms:
            if isinstance(op, PermPivot):
                w = len(op.order)
                p[:, start: start + w] = op.apply_right(p[:, start: start + w])
            elif isinstance(op, ReflPivot):
                w = op.wy.dim
                p[:, start: start + w] = op.apply_right(p[:, start: start + w])
            else:
                w = op.shape[0]
                p[:, start: start + w] = p[:, start: start + w] @ op
        return p

    def perm(self):
        """Composite column permutation (A[:, perm] = A P) for permutation pivots."""
        perm = np.arange(self.n, dtype=np.int64)
        for start, op in self.p_transforms:
            if not isinstance(op, PermPivot):
                raise ValueError("perm() needs permutation pivots")
            perm[start: start + len(op.order)] = perm[start: start + len(op.order)][op.order]
        return perm


def _check_input(a, cfg):
    """blocked.py:152-161."""
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2:
        raise DimensionError("expected a 2-d matrix")
    m, n = a.shape
    if m < n:
        raise DimensionError(f"blocked QR needs rows >= cols, got {m}x{n}")
    if not 1 <= cfg.block <= n:
        raise DimensionError(f"block size must lie in [1, {n}], got {cfg.block}")
    return np.array(a, dtype=np.float64, order="F", copy=True)


def _pivot_for_panel(work, start, b, cfg, rng):
    """blocked.py:164-172."""
    s = cfg.resolved_sketch()
    scfg = SketchConfig(b, s.oversample, s.power, s.orthonormalize_between_powers)
    y = build_sketch(work[start:, start:], scfg, rng)
    if cfg.pivot_kind == "reflectors":
        return select_pivot_reflectors(y, b)
    return select_pivot_permutation(y, b)


def block_qr(a, cfg, rng, inspect=None, max_panels=None):
    """Fig. 4 blocked QR (blocked.py:175-219).

    ``max_panels`` (oracle-only) stops after that many non-final panels; the
    CPU baseline uses it to time a bounded sample of a large factorization.
    """
    work = _check_input(a, cfg)
    m, n = work.shape
    b = cfg.block
    f = Factorization(m, n, b, "reflector_pivot" if cfg.pivot_kind == "reflectors" else "perm_pivot")
    panel = 0
    start = 0
    while start < n:
        panel += 1
        if n - start <= b:
            res = qr_column_pivoted(work[start:, start:])
            work[:start, start:] = work[:start, start:][:, res.perm]
            work[start:, start:] = res.r
            f.q_transforms.append((start, res.q, None))
            f.p_transforms.append((start, PermPivot(res.perm)))
            if inspect is not None:
                inspect(panel, work.copy())
            break
        if max_panels is not None and panel > max_panels:
            break
        pivot = _pivot_for_panel(work, start, b, cfg, rng)
        work[:, start:] = pivot.apply_right(work[:, start:])
        res = qr_tall_pivoted(work[start:, start: start + b])
        work[:start, start: start + b] = work[:start, start: start + b][:, res.perm]
        work[start:, start: start + b] = res.r
        work[start:, start + b:] = apply_wy_left(res.q, work[start:, start + b:], transposed=True)
        f.q_transforms.append((start, res.q, None))
        f.p_transforms.append((start, pivot))
        f.p_transforms.append((start, PermPivot(res.perm)))
        if inspect is not None:
            inspect(panel, work.copy())
        start += b
    f.r = work
    return f


def block_qr_downdate(a, cfg, rng, form="pre"):
    """HQRRP downdated-sketch variant of block_qr (NOT in the reference package).

    Oracle for the B200 ``sketch="downdate"`` mode, restating the HQRRP
    downdate (Martinsson et al., SURVEY §8 "Two sketch modes"): G = Omega^T
    is drawn once (gaussian_matrix(m, b+p), counter += m(b+p)), Y = G A, and
    after each panel Y2 <- Y2 - G1 R12 with G1 = Y1 R11^{-1}, the sketch
    columns following every column move.  Pivot selection, the two-stage panel
    and the trailing update are those of block_qr (blocked.py:175-219).

    The downdate is evaluated in its pre-rotation form, as the B200 driver does
    (driver.cu form_g1): with the panel's unpivoted R' (first stage of
    qr_tall_pivoted), R11 = Q2^T R'11 P-hat and R12 = Q2^T R'12, so
    G1 R12 = Y1' R'11^{-1} R'12 with Y1' the selected sketch columns before
    P-hat -- the same product without Q2 or P-hat (they agree in exact
    arithmetic; this restatement fixes the rounding the GPU path follows).

    ``form="post"`` is the independent restatement of SURVEY section 8's derivation, in the
    order it is written there: P-hat is applied to the sketch columns too, G1 = Y1 R11^{-1}
    with the FINAL R11 (after the b x b CPQR), and Y2 -= G1 R12 with the final R12 (the top
    b rows after the trailing update).  It shares no evaluation order with the GPU path.
    """
    from scipy.linalg import solve_triangular

    work = _check_input(a, cfg)
    m, n = work.shape
    b = cfg.block
    s_cfg = cfg.resolved_sketch()
    wdt = b + s_cfg.oversample
    f = Factorization(m, n, b, "perm_pivot")
    yt = None
    if n > b:
        omega = gaussian_matrix(m, wdt, rng)
        yt = omega.T @ work
    start = 0
    while start < n:
        if n - start <= b:
            res = qr_column_pivoted(work[start:, start:])
            work[:start, start:] = work[:start, start:][:, res.perm]
            work[start:, start:] = res.r
            f.q_transforms.append((start, res.q, None))
            f.p_transforms.append((start, PermPivot(res.perm)))
            break
        if wdt > n - start:
            raise ValueError(f"sketch width {wdt} exceeds the {n - start} columns being pivoted")
        pivot = select_pivot_permutation(yt[:, start:].T, b)
        work[:, start:] = pivot.apply_right(work[:, start:])
        yt[:, start:] = yt[:, start:][:, pivot.order]
        if form == "post":
            res = qr_tall_pivoted(work[start:, start: start + b])
            work[:start, start: start + b] = work[:start, start: start + b][:, res.perm]
            work[start:, start: start + b] = res.r
            work[start:, start + b:] = apply_wy_left(res.q, work[start:, start + b:], transposed=True)
            y1 = yt[:, start: start + b][:, res.perm]
            r11 = res.r[:b, :b]
            g1 = solve_triangular(r11.T, y1.T, lower=True).T  # G1 = Y1 R11^{-1}
            yt[:, start + b:] -= g1 @ work[start: start + b, start + b:]
            f.q_transforms.append((start, res.q, None))
            f.p_transforms.append((start, pivot))
            f.p_transforms.append((start, PermPivot(res.perm)))
            start += b
            continue
        # G1' = Y1' R'11^{-1} from the unpivoted first stage (see the docstring)
        first = qr_unpivoted(work[start:, start: start + b])
        g1 = solve_triangular(first.r[:b, :b].T, yt[:, start: start + b].T, lower=True).T
        a2 = work[start:, start + b:].copy()
        res = qr_tall_pivoted(work[start:, start: start + b])
        work[:start, start: start + b] = work[:start, start: start + b][:, res.perm]
        work[start:, start: start + b] = res.r
        work[start:, start + b:] = apply_wy_left(res.q, work[start:, start + b:], transposed=True)
        r12p = apply_wy_left(wy_accumulate(first.refl, work.shape[0] - start), a2, transposed=True)[:b]  # R'12
        yt[:, start + b:] -= g1 @ r12p
        f.q_transforms.append((start, res.q, None))
        f.p_transforms.append((start, pivot))
        f.p_transforms.append((start, PermPivot(res.perm)))
        start += b
    f.r = work
    return f


def panel_svd(panel):
    """Unpivoted QR then Jacobi SVD of the triangle (blocked.py:222-236); returns (wy, u', d, v)."""
    panel = np.asarray(panel, dtype=np.float64)
    mp, b = panel.shape
    if mp < b:
        raise DimensionError(f"panel must be tall, got {mp}x{b}")
    qr = qr_unpivoted(panel)
    u, d, v = svd_full(qr.r[:b, :])
    return qr.q, u, d, v


def block_rrqr(a, cfg, rng, inspect=None):
    """Fig. 7 rank-revealing variant (blocked.py:239-279)."""
    work = _check_input(a, cfg)
    m, n = work.shape
    b = cfg.block
    cfg = BlockConfig(b, cfg.resolved_sketch(), "reflectors", True)
    f = Factorization(m, n, b, "rrqr")
    panel = 0
    start = 0
    while start < n:
        width = min(b, n - start)
        panel += 1
        final = n - start <= b
        if not final:
            pivot = _pivot_for_panel(work, start, b, cfg, rng)
            work[:, start:] = pivot.apply_right(work[:, start:])
            f.p_transforms.append((start, pivot))
        wy, small, d, v = panel_svd(work[start:, start: start + width])
        work[:start, start: start + width] = work[:start, start: start + width] @ v
        blk = np.zeros((m - start, width), order="F")
        np.fill_diagonal(blk, d)
        work[start:, start: start + width] = blk
        if not final:
            tail = apply_wy_left(wy, work[start:, start + width:], transposed=True)
            tail[:width, :] = small.T @ tail[:width, :]
            work[start:, start + width:] = tail
        f.q_transforms.append((start, wy, small))
        f.p_transforms.append((start, v))
        if inspect is not None:
            inspect(panel, work.copy())
        start += width
    f.r = work
    return f


# --------------------------------------------------------------------------
# Input generators used by the BASELINE configs (matrices.py:34-48)
# --------------------------------------------------------------------------
def haar_orthonormal(n, rng):
    """QR of a Gaussian with the sign fix (matrices.py:34-41)."""
    g = gaussian_matrix(n, n, rng)
    res = qr_unpivoted(g)
    q = apply_wy_left(res.q, np.eye(n, order="F"))
    s = np.sign(np.diag(res.r))
    s[s == 0] = 1.0
    return q * s
