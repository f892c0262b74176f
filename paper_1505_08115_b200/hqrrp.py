"""Host-side mirror of the reference's HQRRP entry points on the B200 library.

Same names, argument meaning and error behaviour as ``randqr``:

* ``block_qr(a, cfg, rng, inspect=None)``   -- blocked.py:175-219
* ``block_rrqr(a, cfg, rng, inspect=None)`` -- blocked.py:239-279
* ``BlockConfig`` / ``SketchConfig`` / ``RngState``  -- blocked.py:42-50,
  pivoting.py:28-51, rng.py:21-26
* ``Factorization`` with ``.r``, ``.expand_q(cols=None)``, ``.expand_p()``
  (blocked.py:122-149), plus ``.perm`` (A[:, perm] = A P).

Every numeric step runs in librandqr_b200.so on the GPU; this module only
converts arrays, validates like the reference and maps return codes onto the
reference's exceptions.  PyTorch is used to own device memory and streams.
"""

from __future__ import annotations

import ctypes
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import DimensionError, check


# --------------------------------------------------------------------------
# Configuration and RNG state (same fields and defaults as the reference)
# --------------------------------------------------------------------------
@dataclass
class RngState:
    """Seed plus the index of the next normal draw (rng.py:21-26)."""

    seed: int
    counter: int = 0


@dataclass
class SketchConfig:
    """Sketch width block+oversample, power iterations, stabilisation (pivoting.py:28-51)."""

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
class BlockConfig:
    """blocked.py:42-50."""

    block: int
    sketch: SketchConfig | None = None
    pivot_kind: str = "permutation"
    rrqr: bool = False

    def resolved_sketch(self):
        return self.sketch if self.sketch is not None else SketchConfig(block=self.block)


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_1505_08115_b200 needs a CUDA device (B200, sm_100a); there is no CPU path")
    return torch


# --------------------------------------------------------------------------
# Engine: one library context (workspace, stream, stored factors)
# --------------------------------------------------------------------------
class Engine:
    """Owns an ``rq_ctx``: device workspace, the CUDA stream, stored factors."""

    def __init__(self, device=None, stream=None):
        torch = _torch()
        self.lib = _lib.load()
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        h = ctypes.c_void_p()
        check(self.lib.rq_ctx_create(ctypes.byref(h), self.device.index, ctypes.c_void_p(self.stream.cuda_stream)))
        self.handle = h
        self._cb = None
        self._owner = None  # weakref to the Factorization whose factors the context holds

    def _release_factors(self):
        """Before the context overwrites its stored factors: hand them to the Factorization that
        still refers to them (blocked.py:122-149: a Factorization owns its transforms)."""
        owner = self._owner() if self._owner is not None else None
        self._owner = None
        if owner is not None and owner._fset is None:
            h = ctypes.c_void_p()
            check(self.lib.rq_factors_detach(self.handle, ctypes.byref(h)))
            owner._fset = _FactorHandle(self.lib, h)

    def _adopt(self, f):
        self._owner = weakref.ref(f)

    def close(self):
        if getattr(self, "handle", None):
            self.lib.rq_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launches(self):
        return int(self.lib.rq_launch_count(self.handle))

    # ----------------------------------------------------------------------
    def alloc_matrix(self, m, n):
        """Column-major m x n fp64 device matrix with an even leading dimension.

        Returned as (storage tensor of shape (n, ld), ld); element (i, j) is storage[j, i].
        """
        torch = _torch()
        ld = m + (m & 1)
        return torch.empty((max(n, 1), max(ld, 2)), dtype=torch.float64, device=self.device), ld

    def upload(self, a):
        """Host (any array-like) or torch tensor -> padded column-major device copy."""
        torch = _torch()
        if isinstance(a, torch.Tensor):
            t = a.to(device=self.device, dtype=torch.float64)
            m, n = t.shape
            buf, ld = self.alloc_matrix(m, n)
            buf[:n, :m].copy_(t.T)
            return buf, ld, m, n
        a = np.asarray(a, dtype=np.float64)
        m, n = a.shape
        buf, ld = self.alloc_matrix(m, n)
        host = torch.from_numpy(np.ascontiguousarray(a.T))
        buf[:n, :m].copy_(host, non_blocking=False)
        return buf, ld, m, n

    @staticmethod
    def download(buf, m, n):
        """Device column-major storage -> numpy m x n, Fortran order."""
        return np.asfortranarray(buf[:n, :m].cpu().numpy().T)


def _make_config(cfg, rrqr, sketch="fresh"):
    s = cfg.resolved_sketch()
    c = _lib.rq_config()
    c.block = int(cfg.block)
    c.oversample = int(s.oversample)
    c.power = int(s.power)
    c.stabilize = -1 if s.orthonormalize_between_powers is None else int(bool(s.orthonormalize_between_powers))
    c.pivot_kind = _lib.RQ_PIVOT_REFLECTORS if (rrqr or cfg.pivot_kind == "reflectors") else _lib.RQ_PIVOT_PERMUTATION
    c.rrqr = int(bool(rrqr))
    if sketch not in ("fresh", "downdate"):
        raise ValueError(f"sketch must be 'fresh' or 'downdate', not {sketch!r}")
    c.sketch_mode = _lib.RQ_SKETCH_FRESH if sketch == "fresh" else _lib.RQ_SKETCH_DOWNDATE
    return c


def _check_input(a):
    """ndim check of blocked.py:152-155 (the rest is validated in the library)."""
    try:
        import torch

        if isinstance(a, torch.Tensor):
            if a.dim() != 2:
                raise DimensionError("expected a 2-d matrix")
            return a
    except ImportError:
        pass
    arr = np.asarray(a, dtype=np.float64)
    if arr.ndim != 2:
        raise DimensionError("expected a 2-d matrix")
    return arr


# --------------------------------------------------------------------------
# Result object
# --------------------------------------------------------------------------
class _FactorHandle:
    """Owns a detached ``rq_factors`` (rq_factors_detach); frees it with the Factorization."""

    def __init__(self, lib, h):
        self.lib, self.h = lib, h

    def __del__(self):
        try:
            if self.h:
                self.lib.rq_factors_destroy(self.h)
                self.h = None
        except Exception:
            pass


class _PermOrder:
    """PermutationPivot-like op (pivoting.py:55-61): ``order`` of the columns it acts on."""

    def __init__(self, order):
        self.order = order

    def apply_right(self, a):
        return np.array(np.asarray(a)[:, self.order], order="F")


class PermTransform:
    """RightTransform (blocked.py:101-119) of one panel with permutation pivots.

    ``order`` acts on columns ``offset..n-1``: the panel's b selected columns in their final
    order (the sketch's pivot order composed with the panel's inner P-hat), then the rest in
    their previous relative order, as the reference keeps them (pivoting.py:125-128).  The
    reference stores the selection and P-hat as two transforms; their product is this one.
    """

    def __init__(self, offset, order):
        self.offset = int(offset)
        self.op = _PermOrder(order)

    @property
    def order(self):
        return self.op.order

    def right_multiply(self, a):
        out = np.array(a, dtype=np.float64, order="F", copy=True)
        w = len(self.op.order)
        out[:, self.offset:self.offset + w] = out[:, self.offset:self.offset + w][:, self.op.order]
        return out


def panel_orders(perm, offsets):
    """Per-panel PermTransforms from the composite permutation (A[:, perm] = A P).

    After panel i the first s_i + w_i entries of ``perm`` are final; the reference keeps the
    columns it did not select in their previous relative order, so the column order before each
    panel -- and hence each panel's order -- follows from ``perm`` alone.
    """
    perm = np.asarray(perm, dtype=np.int64)
    n = len(perm)
    cur = np.arange(n, dtype=np.int64)  # reference column order before the panel
    out = []
    bounds = list(offsets) + [n]
    for i, s in enumerate(offsets):
        e = bounds[i + 1]
        tail = cur[s:]
        pos = np.empty(n, dtype=np.int64)
        pos[tail] = np.arange(len(tail))
        chosen = perm[s:e]
        mask = np.ones(len(tail), dtype=bool)
        mask[pos[chosen]] = False
        order = np.concatenate([pos[chosen], np.nonzero(mask)[0]])
        out.append(PermTransform(s, order))
        cur = np.concatenate([cur[:s], tail[order]])
    return out


class QPanel:
    """QTransform-like proxy of one panel's left factor U_i = (I - V T V^T) diag(Q2, I) on rows
    offset.. (blocked.py:77-99); the factors stay on the device."""

    def __init__(self, fact, index, offset, count):
        self._f, self.index, self.offset, self.count = fact, index, int(offset), int(count)

    def left_multiply(self, a):
        """U_i @ a (dense expansion helper), on the GPU."""
        return self._f._apply_q(self.index, 1, False, a)

    def left_multiply_transposed(self, a):
        """U_i^T @ a."""
        return self._f._apply_q(self.index, 1, True, a)


class PTransform:
    """RightTransform-like proxy of one orthogonal right factor (reflector pivots: S_i, P-hat_i
    and, for block_rrqr, the panel SVD's V~) on columns offset.. (blocked.py:101-119)."""

    def __init__(self, fact, index, offset, width):
        self._f, self.index, self.offset, self.width = fact, index, int(offset), int(width)

    def right_multiply(self, a):
        return self._f._apply_p(self.index, 1, a)


class Factorization:
    """A P = Q R with Q, P held on the device in compact form (blocked.py:122-149).

    Each Factorization owns its factors: when its Engine factorizes again while this object is
    alive, the factors are detached into it first (rq_factors_detach).
    """

    def __init__(self, engine, m, n, b, method, r_dev, ld, perm_dev):
        self.m, self.n, self.b, self.method = m, n, b, method
        self._engine = engine
        self._r_dev = r_dev
        self._ld = ld
        self._perm_dev = perm_dev
        self._r = None
        self._perm = None
        self._fset = None  # _FactorHandle once detached from the engine
        engine._adopt(self)

    def _fptr(self):
        return self._fset.h if self._fset is not None else None

    @property
    def r(self):
        """m x n upper-trapezoidal R (exact zeros below the diagonal), numpy, F-order."""
        if self._r is None:
            self._r = Engine.download(self._r_dev, self.m, self.n)
        return self._r

    @r.setter
    def r(self, value):
        self._r = value

    @property
    def r_device(self):
        """R as a (storage, ld) pair on the device (column-major)."""
        return self._r_dev, self._ld

    @property
    def perm(self):
        """Composite column permutation: A[:, perm] = A P (permutation pivots only)."""
        if self._perm_dev is None:
            raise ValueError("perm is defined for permutation pivots only")
        if self._perm is None:
            self._perm = self._perm_dev.cpu().numpy().astype(np.int64)
        return self._perm

    def _info(self, which):
        eng = self._engine
        cnt = ctypes.c_int32()
        check(eng.lib.rq_factors_info(eng.handle, self._fptr(), which, 0, None, None, ctypes.byref(cnt)))
        k = cnt.value
        offs = np.zeros(max(k, 1), dtype=np.int64)
        wid = np.zeros(max(k, 1), dtype=np.int32)
        check(eng.lib.rq_factors_info(eng.handle, self._fptr(), which, k, offs.ctypes.data_as(ctypes.c_void_p),
                                      wid.ctypes.data_as(ctypes.c_void_p), ctypes.byref(cnt)))
        return offs[:k], wid[:k]

    @property
    def q_transforms(self):
        """Per-panel left factors, in order (Q = U_1 ... U_L), as device-backed proxies."""
        offs, wid = self._info(0)
        return [QPanel(self, i, o, w) for i, (o, w) in enumerate(zip(offs, wid))]

    @property
    def p_transforms(self):
        """Per-panel right factors, in order (P = P_1 ... P_L)."""
        if self._perm_dev is not None:
            offs, _ = self._info(0)
            return panel_orders(self.perm, offs)
        offs, wid = self._info(1)
        return [PTransform(self, i, o, w) for i, (o, w) in enumerate(zip(offs, wid))]

    def _apply_q(self, first, count, trans, a):
        eng = self._engine
        a = np.asarray(a, dtype=np.float64)
        if a.ndim != 2 or a.shape[0] != self.m:
            raise DimensionError(f"expected {self.m} rows, got shape {a.shape}")
        buf, ld, m, cols = eng.upload(a)
        check(eng.lib.rq_apply_q(eng.handle, self._fptr(), first, count, int(trans), cols,
                                 ctypes.c_void_p(buf.data_ptr()), ld))
        return Engine.download(buf, m, cols)

    def _apply_p(self, first, count, a):
        eng = self._engine
        a = np.asarray(a, dtype=np.float64)
        if a.ndim != 2 or a.shape[1] != self.n:
            raise DimensionError(f"expected {self.n} columns, got shape {a.shape}")
        buf, ld, rows, n = eng.upload(a)
        check(eng.lib.rq_apply_p(eng.handle, self._fptr(), first, count, rows, ctypes.c_void_p(buf.data_ptr()), ld))
        return Engine.download(buf, rows, n)

    def apply_q(self, a, transpose=False):
        """Q @ a (or Q^T @ a) for an m-row array, without forming Q."""
        return self._apply_q(0, len(self._info(0)[0]), transpose, a)

    def expand_q_device(self, cols=None):
        eng = self._engine
        cols = self.n if cols is None else int(cols)
        buf, ld = eng.alloc_matrix(self.m, cols)
        if self._fset is not None:
            check(eng.lib.rq_factors_form_q(eng.handle, self._fset.h, cols, ctypes.c_void_p(buf.data_ptr()), ld))
        else:
            check(eng.lib.rq_form_q(eng.handle, cols, ctypes.c_void_p(buf.data_ptr()), ld))
        return buf, ld

    def expand_q(self, cols=None):
        """Dense Q with orthonormal columns, m x cols (default economy m x n)."""
        cols = self.n if cols is None else int(cols)
        buf, _ = self.expand_q_device(cols)
        return Engine.download(buf, self.m, cols)

    def expand_p(self):
        """Dense orthonormal P, n x n."""
        eng = self._engine
        buf, ld = eng.alloc_matrix(self.n, self.n)
        if self._fset is not None:
            check(eng.lib.rq_factors_form_p(eng.handle, self._fset.h, ctypes.c_void_p(buf.data_ptr()), ld))
        else:
            check(eng.lib.rq_form_p(eng.handle, ctypes.c_void_p(buf.data_ptr()), ld))
        return Engine.download(buf, self.n, self.n)


# --------------------------------------------------------------------------
# Entry points
# --------------------------------------------------------------------------
def _run(a, cfg, rng, inspect, rrqr, engine, sketch="fresh", tf32_update=False):
    torch = _torch()
    a = _check_input(a)
    eng = engine if engine is not None else Engine()
    buf, ld, m, n = eng.upload(a)
    c = _make_config(cfg, rrqr, sketch)
    if tf32_update:
        c.flags |= _lib.RQ_FLAG_TF32_UPDATE
    eng._release_factors()
    counter = ctypes.c_uint64(int(rng.counter))
    perm = None if (rrqr or cfg.pivot_kind == "reflectors") else torch.empty(max(n, 1), dtype=torch.int64,
                                                                               device=eng.device)
    if inspect is not None:
        def _cb(panel, _user):
            host = np.zeros((m, n), order="F")
            check(eng.lib.rq_snapshot(eng.handle, host.ctypes.data_as(ctypes.c_void_p), m))
            inspect(int(panel), host)

        eng._cb = _lib.PANEL_CB(_cb)
        check(eng.lib.rq_ctx_set_inspect(eng.handle, eng._cb, None))
    else:
        eng.lib.rq_ctx_set_inspect(eng.handle, _lib.PANEL_CB(), None)
    try:
        rc = eng.lib.rq_factorize(eng.handle, ctypes.byref(c), m, n, ctypes.c_void_p(buf.data_ptr()), ld,
                                  ctypes.c_uint64(int(rng.seed) & 0xFFFFFFFFFFFFFFFF), ctypes.byref(counter),
                                  ctypes.c_void_p(perm.data_ptr()) if perm is not None else None)
        rng.counter = int(counter.value)
        check(rc)
    finally:
        if inspect is not None:
            eng.lib.rq_ctx_set_inspect(eng.handle, _lib.PANEL_CB(), None)
    method = "rrqr" if rrqr else ("reflector_pivot" if cfg.pivot_kind == "reflectors" else "perm_pivot")
    return Factorization(eng, m, n, cfg.block, method, buf, ld, perm)


def block_qr(a, cfg, rng, inspect=None, *, engine=None, sketch="fresh", tf32_update=False):
    """Blocked QR with randomized block pivoting (blocked.py:175-219), on the B200.

    The input is not modified; ``rng.counter`` advances by the draws consumed.
    ``sketch="fresh"`` (default) reproduces the reference: a new Omega per panel.
    ``sketch="downdate"`` is HQRRP proper: G is drawn once (counter += m(b+p)),
    Y = G A is downdated after every panel (Y2 <- Y2 - G1 R12); its pivots
    legitimately differ from the reference's.
    ``tf32_update=True`` is the fp32-accuracy path (BASELINE cfg 3 fp32): the trailing-update
    GEMMs run as 3xTF32 products on the tcgen05 tensor cores (fp32 accumulation) instead of FP64
    DMMA; panels, sketches and pivot selection stay fp64 (RQ_FLAG_TF32_UPDATE).
    """
    return _run(a, cfg, rng, inspect, False, engine, sketch, tf32_update)


def block_rrqr(a, cfg, rng, inspect=None, *, engine=None):
    """Rank-revealing variant (blocked.py:239-279), on the B200."""
    return _run(a, cfg, rng, inspect, True, engine)


# --------------------------------------------------------------------------
# Kernel-plugin level and RNG
# --------------------------------------------------------------------------
def householder_sweep(a, v, perm, steps, pivot, *, engine=None):
    """In-place ``householder_sweep(a, v, perm, steps, pivot)`` (_kernels_numpy.py:11-22) on the GPU.

    Numpy arguments are updated in place (round trip through device memory);
    torch CUDA tensors (column-major storage) are used as they are.
    """
    torch = _torch()
    eng = engine if engine is not None else Engine()
    a_np = np.asarray(a)
    m, n = a_np.shape
    abuf, lda, _, _ = eng.upload(a_np)
    vbuf, ldv = eng.alloc_matrix(m, max(steps, 1))
    vbuf.zero_()
    pt = torch.from_numpy(np.asarray(perm, dtype=np.int64).copy()).to(eng.device)
    check(eng.lib.rq_householder_sweep(eng.handle, ctypes.c_void_p(abuf.data_ptr()), m, n, lda,
                                       ctypes.c_void_p(vbuf.data_ptr()), ldv, ctypes.c_void_p(pt.data_ptr()),
                                       int(steps), int(bool(pivot))))
    a[...] = Engine.download(abuf, m, n)
    if steps > 0:
        v[:, :steps] = Engine.download(vbuf, m, steps)
    perm[...] = pt.cpu().numpy()


def gaussian_matrix_device(rows, cols, rng, *, engine=None):
    """gaussian_matrix (rng.py:54-68) generated on the GPU; returns (storage, ld)."""
    if rows < 1 or cols < 1:
        raise DimensionError(f"matrix dimensions must be positive, got {rows}x{cols}")
    eng = engine if engine is not None else Engine()
    buf, ld = eng.alloc_matrix(rows, cols)
    check(eng.lib.rq_gaussian_matrix(eng.handle, rows, cols, int(rng.seed) & 0xFFFFFFFFFFFFFFFF, int(rng.counter),
                                     ctypes.c_void_p(buf.data_ptr()), ld))
    rng.counter += rows * cols
    return buf, ld


def gaussian_matrix(rows, cols, rng, *, engine=None):
    """gaussian_matrix (rng.py:54-68): column-major, counter advances by rows*cols."""
    buf, _ = gaussian_matrix_device(rows, cols, rng, engine=engine)
    return Engine.download(buf, rows, cols)


def splitmix_words(seed, first, count, *, engine=None):
    """Raw splitmix64 words (rng.py:29-39) computed on the GPU."""
    torch = _torch()
    eng = engine if engine is not None else Engine()
    out = torch.empty(max(count, 1), dtype=torch.int64, device=eng.device)
    check(eng.lib.rq_splitmix_words(eng.handle, int(seed) & 0xFFFFFFFFFFFFFFFF, int(first), int(count),
                                    ctypes.c_void_p(out.data_ptr())))
    return out[:count].cpu().numpy().view(np.uint64)
