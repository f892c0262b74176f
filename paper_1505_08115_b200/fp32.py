"""fp32 path (BASELINE cfg 3 "fp32 and fp64").

Two drivers: ``block_qr_fp32(..., driver="monolithic")`` (default on one GPU) runs the C++
driver with RQ_FLAG_TF32_UPDATE -- the trailing-update GEMMs, the dominant flops, as 3xTF32
products on the tcgen05 tensor cores, panels / sketches / pivots in fp64; the panel-step engine
below keeps A itself in fp32 (half the bytes; process groups).

The reference is fp64-only (blocked.py:161 converts its input), so this is an
extension with its own accuracy bar (north star: ||AP - QR|| / ||A|| and
||Q^T Q - I|| <= 1e-5) and with the pivots compared against the fp64 path where the
spectrum is well separated.

Mixed precision, by where the work is:
* A stays fp32 in HBM (half the bytes of the fp64 path).  The sketch Y = Omega^T X, the
  trailing update A2 <- (I - V T V^T)^T A2 with its top rows <- Q2^T, and the formation of Q
  run on this library's fp32 tensor-core GEMM (rq_gemm_f32: 3xTF32 split products on
  tcgen05.mma, TMA staging, TMEM accumulator -- csrc/gemm_tf32.cu);
* the latency-bound serial kernels -- sketch CPQR (pivot choice), panel leaf QR, b x b
  CPQR, T -- run in this library's fp64 kernels on fp64 copies of Y and of the panel
  (rq_sketch_select, rq_panel_factor, rq_householder_sweep), and their factors are
  rounded to fp32 for the GEMMs.

The panel loop is dist.factorize_local with this engine at world size 1 (or over a
process group: the fp32 path shards the same way as the fp64 one).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from .dist import CudaStepEngine, factorize_local, gather_r
from .errors import check
from .hqrrp import BlockConfig, Engine, RngState


def _p(t, off=0):
    return ctypes.c_void_p(t.data_ptr() + 4 * off)


class Fp32StepEngine:
    """fp32 storage and tensor-core GEMMs; fp64 serial kernels on converted copies."""

    ld_align = 4  # rq_gemm_f32: ld % 4 == 0, 16-byte aligned operand bases
    defer_rest = CudaStepEngine.defer_rest

    def __init__(self, engine: Engine | None = None, keep_factors: bool = False):
        import torch

        self.torch = torch
        self.f64 = CudaStepEngine(engine)
        self.lib = self.f64.lib
        self.h = self.f64.h
        self.device = self.f64.device
        self.keep = keep_factors
        self.panels = []  # (s, mp, b, (v, ldv, t, ldt, q2, ldq)) when keep_factors
        self.final = None  # (s, mp, w, v (fp32), ldv) of the final block's reflectors

    def alloc(self, rows, cols):
        torch = self.torch
        ld = (rows + 3) // 4 * 4
        return torch.zeros((max(cols, 1), max(ld, 4)), dtype=torch.float32, device=self.device), ld

    def gemm(self, mmajor, M, N, K, a, lda, a_rows, a_cols, a_r0, a_c0, b, ldb, b_rows, b_cols, b_r0, b_c0, c, ldc,
             c_off, alpha, beta, h=None):
        """rq_gemm_f32 on (cols, ld) storages; c_off = element offset of C's view."""
        if M <= 0 or N <= 0:
            return
        check(self.lib.rq_gemm_f32(h or self.h, int(mmajor), M, N, K, _p(a), lda, a_rows, a_cols, a_r0, a_c0, _p(b),
                                   ldb, b_rows, b_cols, b_r0, b_c0, _p(c, c_off), ldc, float(alpha), float(beta)))

    def shifted(self, x, ldx, rows, cols, r0):
        """x (rows x cols) re-based at row r0 % 4 of a new buffer: a TN product's two K origins must
        agree mod 4 (16-byte TMA origins); returns (buffer, ld, row origin)."""
        off = r0 % 4
        if off == 0:
            return x, ldx, 0
        y, ldy = self.alloc(rows + off, cols)
        y[:cols, off:off + rows] = x[:cols, :rows]
        return y, ldy, off

    def gaussian(self, rows, cols, seed, counter):
        g, _ = self.f64.gaussian(rows, cols, seed, counter)  # the reference's fp64 draws
        out, ld = self.alloc(rows, cols)
        out[:cols, :rows] = g[:cols, :rows]
        return out, ld

    # storage convention: (cols, ld) tensor, row j of the storage = column j of the matrix
    def sketch(self, om, ldo, a, lda, a_rows, a_cols, r0, c0, mp, nt, wdt, cols_alloc):
        y, ldy = self.alloc(wdt, max(cols_alloc, 1))
        if nt > 0:  # Y^T = Omega^T X (TN)
            o, ldo2, oo = self.shifted(om, ldo, mp, wdt, r0)
            self.gemm(0, wdt, nt, mp, o, ldo2, mp + oo, wdt, oo, 0, a, lda, a_rows, a_cols, r0, c0, y, ldy, 0, 1.0,
                      0.0)
        return y, ldy

    def index(self, arr):
        return self.f64.index(arr)

    def select_async(self, y, ldy, wdt, n, steps, init_pos):
        y64, ld64 = self.f64.alloc(wdt, n)
        y64[:n, :wdt] = y[:n, :wdt]
        return self.f64.select_async(y64, ld64, wdt, n, steps, init_pos)

    def select(self, y, ldy, wdt, n, steps, init_pos):
        return self.select_async(y, ldy, wdt, n, steps, init_pos).result()

    def panel_factor(self, p, ldp, mp, b):
        p64, ldp64 = self.f64.alloc(mp, b)
        p64[:b, :mp] = p[:b, :mp]
        (v, ldv, t, ldt, q2, ldq), ph = self.f64.panel_factor(p64, ldp64, mp, b)
        p[:b, :mp] = p64[:b, :mp]
        v32, ldv32 = self.alloc(mp, b)
        v32[:b, :mp] = v[:b, :mp]
        t32, ldt32 = self.alloc(b, b)
        t32[:b, :b] = t[:b, :b]
        q32, ldq32 = self.alloc(b, b)
        q32[:b, :b] = q2[:b, :b]
        return (v32, ldv32, t32, ldt32, q32, ldq32), ph

    def panel_apply(self, fac, mp, b, a, lda, a_rows, a_cols, r0, c0, n2):
        """A2 <- (I - V T V^T)^T A2, top b rows <- Q2^T top (rq_panel_apply in fp32)."""
        v, ldv, t, ldt, q2, ldq = fac
        w, ldw = self.alloc(b, n2)
        w2, _ = self.alloc(b, n2)
        # W = V^T A2 (TN), W2 = T^T W (TN), A2 -= V W2 (NN)
        vs, ldvs, vo = self.shifted(v, ldv, mp, b, r0)
        self.gemm(0, b, n2, mp, vs, ldvs, mp + vo, b, vo, 0, a, lda, a_rows, a_cols, r0, c0, w, ldw, 0, 1.0, 0.0)
        self.gemm(0, b, n2, b, t, ldt, b, b, 0, 0, w, ldw, b, n2, 0, 0, w2, ldw, 0, 1.0, 0.0)
        self.gemm(1, mp, n2, b, v, ldv, mp, b, 0, 0, w2, ldw, b, n2, 0, 0, a, lda, c0 * lda + r0, -1.0, 1.0)
        # top rows: Q2^T (TN) from a copy
        w[:n2, :b] = a[c0:c0 + n2, r0:r0 + b]
        self.gemm(0, b, n2, b, q2, ldq, b, b, 0, 0, w, ldw, b, n2, 0, 0, a, lda, c0 * lda + r0, 1.0, 0.0)

    def panel_apply_top(self, fac, mp, b, a, lda, a_rows, a_cols, r0, c0, n2):
        """Look-ahead split (dist.factorize_local): W, W2, the top b rows and Q2^T now."""
        v, ldv, t, ldt, q2, ldq = fac
        w, ldw = self.alloc(b, n2)
        w2, _ = self.alloc(b, n2)
        vs, ldvs, vo = self.shifted(v, ldv, mp, b, r0)
        self.gemm(0, b, n2, mp, vs, ldvs, mp + vo, b, vo, 0, a, lda, a_rows, a_cols, r0, c0, w, ldw, 0, 1.0, 0.0)
        self.gemm(0, b, n2, b, t, ldt, b, b, 0, 0, w, ldw, b, n2, 0, 0, w2, ldw, 0, 1.0, 0.0)
        self.gemm(1, b, n2, b, v, ldv, mp, b, 0, 0, w2, ldw, b, n2, 0, 0, a, lda, c0 * lda + r0, -1.0, 1.0)
        w[:n2, :b] = a[c0:c0 + n2, r0:r0 + b]
        self.gemm(0, b, n2, b, q2, ldq, b, b, 0, 0, w, ldw, b, n2, 0, 0, a, lda, c0 * lda + r0, 1.0, 0.0)
        return w2, ldw

    def panel_apply_rest(self, fac, top, mp, b, a, lda, a_rows, a_cols, r0, c0, n2, w_off=0, h=None):
        v, ldv, t, ldt, q2, ldq = fac
        w2, ldw = top
        if mp > b and n2 > 0:
            self.gemm(1, mp - b, n2, b, v, ldv, mp, b, b, 0, w2, ldw, b, w2.shape[0], 0, w_off, a, lda,
                      c0 * lda + r0 + b, -1.0, 1.0, h=h)

    def panel_apply_rest_cols(self, fac, top, mp, b, a, lda, r0, t1, cols):
        """The deferred rest of the update on the listed local columns (gathered), then their
        W2 columns zeroed (dist.factorize_local's look-ahead)."""
        if mp <= b or len(cols) == 0:
            return
        w2, ldw = top
        idx = self.index(cols)
        widx = self.index(np.asarray(cols) - t1)
        k = len(cols)
        x, ldx = self.alloc(mp - b, k)
        x[:k, :mp - b] = a.index_select(0, idx)[:, r0 + b:r0 + mp]
        ws, ldws = self.alloc(b, k)
        ws[:k, :b] = w2.index_select(0, widx)[:, :b]
        v, ldv = fac[0], fac[1]
        self.gemm(1, mp - b, k, b, v, ldv, mp, b, b, 0, ws, ldws, b, k, 0, 0, x, ldx, 0, -1.0, 1.0)
        rows = a.index_select(0, idx)
        rows[:, r0 + b:r0 + mp] = x[:k, :mp - b]
        a.index_copy_(0, idx, rows)
        w2.index_fill_(0, widx, 0.0)

    def zero_cols(self, top, cols):
        self.f64.zero_cols(top, cols)

    def rest_async(self, fac, top, mp, b, a, lda, a_rows, a_cols, r0, c0, n2, w_off, keep):
        torch = self.torch
        se = self.f64._side()
        ev0 = torch.cuda.Event()
        ev0.record(self.f64.eng.stream)
        se.stream.wait_event(ev0)
        with torch.cuda.stream(se.stream):
            self.panel_apply_rest(fac, top, mp, b, a, lda, a_rows, a_cols, r0, c0, n2, w_off, h=se.handle)
            for t in keep:
                t.record_stream(se.stream)
            top[0].record_stream(se.stream)
        ev1 = torch.cuda.Event()
        ev1.record(se.stream)
        return ev1

    def wait(self, ev):
        self.f64.wait(ev)

    def downdate_g1(self, y, ldy, wdt, c0, ph, p, ldp, b, g1, ldg):
        """G1 = Y1 R11^{-1} in fp64 (the serial kernels), rounded to fp32 for the downdate GEMM."""
        y64, ldy64 = self.f64.alloc(wdt, b)
        y64[:b, :wdt] = y[c0:c0 + b, :wdt]
        p64, ldp64 = self.f64.alloc(b, b)
        p64[:b, :b] = p[:b, :b]
        g64, ldg64 = self.f64.alloc(wdt, b)
        self.f64.downdate_g1(y64, ldy64, wdt, 0, ph, p64, ldp64, b, g64, ldg64)
        g1[:b, :wdt] = g64[:b, :wdt]

    def downdate_apply(self, g1, ldg, wdt, b, a, lda, a_rows, a_cols, s, t1, n2, y, ldy):
        """Y2 <- Y2 - G1 R12 on the local columns t1 .. t1+n2 (fp32, NN)."""
        if n2 <= 0:
            return
        self.gemm(1, wdt, n2, b, g1, ldg, wdt, b, 0, 0, a, lda, a_rows, a_cols, s, t1, y, ldy, t1 * ldy, -1.0, 1.0)

    def record_panel(self, s, mp, b, fac):
        if self.keep:
            self.panels.append((s, mp, b, fac))

    def final_block(self, blk, ldb, mp, w):
        b64, ld64 = self.f64.alloc(mp, w)
        b64[:w, :mp] = blk[:w, :mp]
        torch = self.torch
        v, ldv = self.f64.alloc(mp, w)
        perm = torch.arange(w, dtype=torch.int64, device=self.device)
        check(self.lib.rq_householder_sweep(self.h, ctypes.c_void_p(b64.data_ptr()), mp, w, ld64,
                                            ctypes.c_void_p(v.data_ptr()), ldv, ctypes.c_void_p(perm.data_ptr()),
                                            min(mp, w), 1))
        blk[:w, :mp] = b64[:w, :mp]
        if self.keep:
            v32, ldv32 = self.alloc(mp, w)
            v32[:w, :mp] = v[:w, :mp]
            self.final = (mp, min(mp, w), v32, ldv32)
        return perm

    def form_q(self, m, cols):
        """Q (m x cols, fp32 storage) = U_1 ... U_L H_final applied to I on the tensor cores
        (Factorization.expand_q, blocked.py:134-141).  Needs keep_factors=True at world size 1."""
        q, ldq = self.alloc(m, cols)
        q[:cols, :cols] = self.torch.eye(cols, dtype=self.torch.float32, device=self.device)
        bmax = max([b for _, _, b, _ in self.panels] + [1])
        w_, ldw = self.alloc(bmax, cols)
        w2, _ = self.alloc(bmax, cols)
        tmp, _ = self.alloc(bmax, cols)
        if self.final is not None:
            mp, k, v, ldv = self.final
            s = m - mp
            vs, ldvs, vo = self.shifted(v, ldv, mp, k, s)
            for j in range(k - 1, -1, -1):  # H_j = I - 2 u_j u_j^T on rows s..
                self.gemm(0, 1, cols, mp, vs, ldvs, mp + vo, k, vo, j, q, ldq, m, cols, s, 0, w_, ldw, 0, 1.0, 0.0)
                self.gemm(1, mp, cols, 1, v, ldv, mp, k, 0, j, w_, ldw, 1, cols, 0, 0, q, ldq, s, -2.0, 1.0)
        for s, mp, b, (v, ldv, t, ldt, q2, ldq2) in reversed(self.panels):
            # X[0:b] <- Q2 X[0:b] (NN), then X <- X - V T (V^T X)
            tmp[:cols, :b] = q[:cols, s:s + b]
            self.gemm(1, b, cols, b, q2, ldq2, b, b, 0, 0, tmp, ldw, b, cols, 0, 0, q, ldq, s, 1.0, 0.0)
            vs, ldvs, vo = self.shifted(v, ldv, mp, b, s)
            self.gemm(0, b, cols, mp, vs, ldvs, mp + vo, b, vo, 0, q, ldq, m, cols, s, 0, w_, ldw, 0, 1.0, 0.0)
            self.gemm(1, b, cols, b, t, ldt, b, b, 0, 0, w_, ldw, b, cols, 0, 0, w2, ldw, 0, 1.0, 0.0)
            self.gemm(1, mp, cols, b, v, ldv, mp, b, 0, 0, w2, ldw, b, cols, 0, 0, q, ldq, s, -1.0, 1.0)
        return q, ldq

    def synchronize(self):
        self.f64.synchronize()


@dataclass
class Fp32Result:
    r: np.ndarray     # m x n upper trapezoidal, float32
    perm: np.ndarray  # A[:, perm] = Q R
    q: np.ndarray | None = None  # m x n float32 (economy Q) when requested


def block_qr_fp32(a, cfg: BlockConfig, rng: RngState, *, engine=None, group=None, want_q=False, sketch="fresh",
                  driver=None):
    """block_qr (blocked.py:175) at fp32 accuracy.  ``rng.counter`` advances exactly as in the
    fp64 / reference run.  want_q: also form the economy Q (fp32).

    driver="monolithic" (default on one GPU): the C++ driver with RQ_FLAG_TF32_UPDATE -- the
    trailing-update GEMMs on the tcgen05 tensor cores (3xTF32), everything else fp64;
    driver="steps" (default with a process group): fp32 storage through the panel-step driver."""
    import torch

    if driver is None:
        driver = "steps" if group is not None else "monolithic"
    if driver == "monolithic":
        from .hqrrp import block_qr

        f = block_qr(np.asarray(a, dtype=np.float64), cfg, rng, engine=engine, sketch=sketch, tf32_update=True)
        q = f.expand_q().astype(np.float32) if want_q else None
        return Fp32Result(np.asfortranarray(f.r.astype(np.float32)), f.perm, q)
    eng = Fp32StepEngine(engine, keep_factors=want_q)
    a = np.asarray(a, dtype=np.float32)
    m, n = a.shape
    buf, ld = eng.alloc(m, n)
    buf[:n, :m] = torch.from_numpy(np.ascontiguousarray(a.T)).to(eng.device)
    res = factorize_local(buf, ld, m, n, cfg, rng, group=group, engine=eng, sketch=sketch)
    r_full = gather_r(res, eng, group)
    r = np.asfortranarray(r_full[:n, :m].cpu().numpy().T)
    q = None
    if want_q:
        qs, _ = eng.form_q(m, n)
        q = np.asfortranarray(qs[:n, :m].cpu().numpy().T)
    return Fp32Result(np.triu(r), res.perm, q)
