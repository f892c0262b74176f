"""CPU stand-in for dist.CudaStepEngine, used only by the multi-process (gloo) tests.

TEST INFRASTRUCTURE: each panel step is computed with the oracle (oracle/randqr_oracle.py,
the CPU restatement of the reference), so the gloo tests check the distributed
orchestration of paper_1505_08115_b200/dist.py -- block-cyclic ownership, the
all-gather, the column exchange, the broadcast of the panel factors and the
replicated bookkeeping -- against the single-process reference algorithm.  The
product path never imports this module; the CUDA engine's steps are checked
against the monolithic GPU driver in tests/test_gpu_dist.py.

The step semantics are those of the C ABI's panel-step entry points
(include/randqr_b200.h: rq_sketch_select, rq_panel_factor, rq_panel_apply):
reflectors H = I - 2 u u^T (householder.py:55-69), T = (I/2 + striu(V^T V))^{-1},
qr_tall_pivoted = unpivoted QR + CPQR of R' (householder.py:183-198).
"""

import os
import sys

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(_HERE, "..", "oracle"))
import randqr_oracle as orc  # noqa: E402


def _tfac(v):
    k = v.shape[1]
    return np.linalg.inv(0.5 * np.eye(k) + np.triu(v.T @ v, 1))


class NumpyStepEngine:
    torch = torch
    defer_rest = True  # exercise dist.factorize_local's deferred-update bookkeeping

    def __init__(self):
        self.device = torch.device("cpu")

    def alloc(self, rows, cols):
        ld = rows + (rows & 1)
        return torch.zeros((max(cols, 1), max(ld, 2)), dtype=torch.float64), ld

    @staticmethod
    def _get(buf, rows, cols, r0=0, c0=0):
        return np.asfortranarray(buf[c0:c0 + cols, r0:r0 + rows].numpy().T)

    @staticmethod
    def _put(buf, x, r0=0, c0=0):
        rows, cols = x.shape
        buf[c0:c0 + cols, r0:r0 + rows] = torch.from_numpy(np.ascontiguousarray(x.T))

    def gaussian(self, rows, cols, seed, counter):
        buf, ld = self.alloc(rows, cols)
        self._put(buf, orc.gaussian_matrix(rows, cols, orc.RngState(seed, counter)))
        return buf, ld

    def sketch(self, om, ldo, a, lda, a_rows, a_cols, r0, c0, mp, nt, wdt, cols_alloc):
        y, ldy = self.alloc(wdt, max(cols_alloc, 1))
        if nt > 0:
            omega = self._get(om, mp, wdt)
            x = self._get(a, mp, nt, r0, c0)
            self._put(y, omega.T @ x)
        return y, ldy

    def select(self, y, ldy, wdt, n, steps, init_pos):
        ymat = self._get(y, wdt, n)
        order = np.argsort(np.asarray(init_pos), kind="stable")
        yo = np.asfortranarray(ymat[:, order])
        v = np.zeros((wdt, steps), order="F")
        perm = np.arange(n, dtype=np.int64)
        orc.householder_sweep(yo, v, perm, steps, True)
        return order[perm[:steps]].astype(np.int64)

    def panel_factor(self, p, ldp, mp, b):
        pm = self._get(p, mp, b)
        v = np.zeros((mp, b), order="F")
        orc.householder_sweep(pm, v, np.arange(b, dtype=np.int64), b, False)
        s = np.asfortranarray(np.triu(pm[:b, :b]))
        v2 = np.zeros((b, b), order="F")
        ph = np.arange(b, dtype=np.int64)
        orc.householder_sweep(s, v2, ph, b, True)
        q2 = np.eye(b) - v2 @ _tfac(v2) @ v2.T
        out = np.zeros((mp, b))
        out[:b] = np.triu(s)
        self._put(p, out)
        vb, ldv = self.alloc(mp, b)
        self._put(vb, v)
        tb, ldt = self.alloc(b, b)
        self._put(tb, _tfac(v))
        qb, ldq = self.alloc(b, b)
        self._put(qb, q2)
        return (vb, ldv, tb, ldt, qb, ldq), torch.from_numpy(ph)

    def panel_apply(self, fac, mp, b, a, lda, a_rows, a_cols, r0, c0, n2):
        vb, ldv, tb, ldt, qb, ldq = fac
        v = self._get(vb, mp, b)
        t = self._get(tb, b, b)
        q2 = self._get(qb, b, b)
        x = self._get(a, mp, n2, r0, c0)
        x -= v @ (t.T @ (v.T @ x))
        x[:b] = q2.T @ x[:b]
        self._put(a, x, r0, c0)

    def panel_apply_top(self, fac, mp, b, a, lda, a_rows, a_cols, r0, c0, n2):
        """Look-ahead split of panel_apply: the top b rows now (W2 returned), the rest later."""
        vb, ldv, tb, ldt, qb, ldq = fac
        v = self._get(vb, mp, b)
        t = self._get(tb, b, b)
        q2 = self._get(qb, b, b)
        x = self._get(a, mp, n2, r0, c0)
        w2 = t.T @ (v.T @ x)
        top = x[:b] - v[:b] @ w2
        self._put(a, q2.T @ top, r0, c0)
        return w2

    def panel_apply_rest(self, fac, w2, mp, b, a, lda, a_rows, a_cols, r0, c0, n2, w_off=0):
        vb = fac[0]
        v = self._get(vb, mp, b)
        if mp > b and n2 > 0:
            x = self._get(a, mp - b, n2, r0 + b, c0)
            self._put(a, x - v[b:] @ w2[:, w_off:w_off + n2], r0 + b, c0)

    # deferred-rest protocol of dist.factorize_local (synchronous here: exercises the
    # column bookkeeping of the look-ahead on CPU)
    def panel_apply_rest_cols(self, fac, w2, mp, b, a, lda, r0, t1, cols):
        v = self._get(fac[0], mp, b)
        for c in cols:
            if mp > b:
                x = self._get(a, mp - b, 1, r0 + b, c)
                self._put(a, x - v[b:] @ w2[:, c - t1:c - t1 + 1], r0 + b, c)
            w2[:, c - t1] = 0.0

    def zero_cols(self, w2, cols):
        for c in cols:
            w2[:, c] = 0.0

    def rest_async(self, fac, w2, mp, b, a, lda, a_rows, a_cols, r0, c0, n2, w_off, keep):
        self.panel_apply_rest(fac, w2, mp, b, a, lda, a_rows, a_cols, r0, c0, n2, w_off)
        return None

    def wait(self, ev):
        pass

    def downdate_g1(self, y, ldy, wdt, c0, ph, p, ldp, b, g1, ldg):
        y1 = self._get(y, wdt, b, 0, c0)[:, np.asarray(ph, dtype=np.int64)]
        r11 = np.triu(self._get(p, b, b))
        self._put(g1, np.linalg.solve(r11.T, y1.T).T)  # Y1 R11^{-1}

    def downdate_apply(self, g1, ldg, wdt, b, a, lda, a_rows, a_cols, s, t1, n2, y, ldy):
        if n2 <= 0:
            return
        g = self._get(g1, wdt, b)
        r12 = self._get(a, b, n2, s, t1)
        yy = self._get(y, wdt, n2, 0, t1)
        self._put(y, yy - g @ r12, 0, t1)

    def final_block(self, blk, ldb, mp, w):
        x = self._get(blk, mp, w)
        v = np.zeros((mp, w), order="F")
        perm = np.arange(w, dtype=np.int64)
        orc.householder_sweep(x, v, perm, min(mp, w), True)
        self._put(blk, x)
        return torch.from_numpy(perm)

    def synchronize(self):
        pass
