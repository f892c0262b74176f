"""fp32 path (BASELINE cfg 3 "fp32 and fp64").

The reference is fp64-only (blocked.py:161 converts its input), so this is an
extension with its own accuracy bar (north star: ||AP - QR|| / ||A|| and
||Q^T Q - I|| <= 1e-5) and with the pivots compared against the fp64 path where the
spectrum is well separated.

Mixed precision, by where the work is:
* A stays fp32 in HBM (half the bytes of the fp64 path); the sketch Y = Omega^T X and
  the trailing update A2 <- (I - V T V^T)^T A2, top rows <- Q2^T, run as fp32 GEMMs
  (cuBLAS SGEMM through torch, TF32 disabled: TF32 alone cannot meet 1e-5);
* the latency-bound serial kernels -- sketch CPQR (pivot choice), panel leaf QR, b x b
  CPQR, T -- run in this library's fp64 kernels on fp64 copies of Y and of the panel
  (rq_sketch_select, rq_panel_factor, rq_householder_sweep), and their factors are
  rounded to fp32 for the GEMMs.

The panel loop is dist.factorize_local with this engine at world size 1 (or over a
process group: the fp32 path shards the same way as the fp64 one).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .dist import CudaStepEngine, factorize_local, gather_r
from .hqrrp import BlockConfig, Engine, RngState


class Fp32StepEngine:
    """fp32 storage and GEMMs; fp64 serial kernels on converted copies."""

    def __init__(self, engine: Engine | None = None):
        import torch

        self.torch = torch
        self.f64 = CudaStepEngine(engine)
        self.device = self.f64.device

    def alloc(self, rows, cols):
        torch = self.torch
        ld = (rows + 3) // 4 * 4
        return torch.zeros((max(cols, 1), max(ld, 4)), dtype=torch.float32, device=self.device), ld

    def _mm(self, x, y):
        torch = self.torch
        saved = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = False
        try:
            return x @ y
        finally:
            torch.backends.cuda.matmul.allow_tf32 = saved

    def gaussian(self, rows, cols, seed, counter):
        g, _ = self.f64.gaussian(rows, cols, seed, counter)  # the reference's fp64 draws
        out, ld = self.alloc(rows, cols)
        out[:cols, :rows] = g[:cols, :rows]
        return out, ld

    # storage convention: (cols, ld) tensor, row j of the storage = column j of the matrix
    def sketch(self, om, ldo, a, lda, a_rows, a_cols, r0, c0, mp, nt, wdt, cols_alloc):
        y, ldy = self.alloc(wdt, max(cols_alloc, 1))
        if nt > 0:
            x_t = a[c0:c0 + nt, r0:r0 + mp]          # X^T (nt x mp)
            y[:nt, :wdt] = self._mm(x_t, om[:wdt, :mp].T)  # Y^T = X^T Omega
        return y, ldy

    def select(self, y, ldy, wdt, n, steps, init_pos):
        y64, ld64 = self.f64.alloc(wdt, n)
        y64[:n, :wdt] = y[:n, :wdt]
        return self.f64.select(y64, ld64, wdt, n, steps, init_pos)

    def panel_factor(self, p, ldp, mp, b):
        p64, ldp64 = self.f64.alloc(mp, b)
        p64[:b, :mp] = p[:b, :mp]
        (v, ldv, t, ldt, q2, ldq), ph = self.f64.panel_factor(p64, ldp64, mp, b)
        p[:b, :mp] = p64[:b, :mp]
        return (v.float(), ldv, t.float(), ldt, q2.float(), ldq), ph

    def panel_apply(self, fac, mp, b, a, lda, a_rows, a_cols, r0, c0, n2):
        v, _, t, _, q2, _ = fac
        vt = v[:b, :mp]              # V^T (b x mp)
        x_t = a[c0:c0 + n2, r0:r0 + mp]  # A2^T (n2 x mp)
        w_t = self._mm(x_t, vt.T)        # W^T = A2^T V            (n2 x b)
        w2_t = self._mm(w_t, t[:b, :b].T)  # W2^T = W^T T          (T(i, j) = t[j, i])
        x_t -= self._mm(w2_t, vt)        # A2^T -= W2^T V^T
        top = x_t[:, :b].clone()
        x_t[:, :b] = self._mm(top, q2[:b, :b].T)  # (Q2^T A2top)^T = A2top^T Q2

    def final_block(self, blk, ldb, mp, w):
        b64, ld64 = self.f64.alloc(mp, w)
        b64[:w, :mp] = blk[:w, :mp]
        perm = self.f64.final_block(b64, ld64, mp, w)
        blk[:w, :mp] = b64[:w, :mp]
        return perm

    def synchronize(self):
        self.f64.synchronize()


@dataclass
class Fp32Result:
    r: np.ndarray     # m x n upper trapezoidal, float32
    perm: np.ndarray  # A[:, perm] = Q R


def block_qr_fp32(a, cfg: BlockConfig, rng: RngState, *, engine=None, group=None):
    """block_qr (blocked.py:175) with A, its sketches and the trailing updates in fp32.
    ``rng.counter`` advances exactly as in the fp64 / reference run."""
    import torch

    eng = Fp32StepEngine(engine)
    a = np.asarray(a, dtype=np.float32)
    m, n = a.shape
    buf, ld = eng.alloc(m, n)
    buf[:n, :m] = torch.from_numpy(np.ascontiguousarray(a.T)).to(eng.device)
    res = factorize_local(buf, ld, m, n, cfg, rng, group=group, engine=eng)
    r_full = gather_r(res, eng, group)
    r = np.asfortranarray(r_full[:n, :m].cpu().numpy().T)
    return Fp32Result(np.triu(r), res.perm)
