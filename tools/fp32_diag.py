"""Diagnostic (not product): fp32 path residuals with the tcgen05 3xTF32 GEMM vs torch SGEMM."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1505_08115_b200 as rq
from paper_1505_08115_b200 import fp32 as F

torch.backends.cuda.matmul.allow_tf32 = False


def torch_gemm(self, mmajor, M, N, K, a, lda, a_rows, a_cols, a_r0, a_c0, b, ldb, b_rows, b_cols, b_r0, b_c0, c, ldc,
               c_off, alpha, beta):
    if M <= 0 or N <= 0:
        return
    A = a.view(-1)[: a_cols * lda].view(a_cols, lda)[:, :a_rows].T  # rows x cols view
    B = b.view(-1)[: b_cols * ldb].view(b_cols, ldb)[:, :b_rows].T
    opa = A[a_r0:a_r0 + M, a_c0:a_c0 + K] if mmajor else A[a_r0:a_r0 + K, a_c0:a_c0 + M].T
    bb = B[b_r0:b_r0 + K, b_c0:b_c0 + N]
    flat = c.view(-1)
    cols = torch.arange(N, device=c.device) * ldc + c_off
    idx = cols[None, :] + torch.arange(M, device=c.device)[:, None]
    cur = flat[idx]
    flat[idx] = (alpha * (opa @ bb) + (beta * cur if beta != 0 else 0)).to(torch.float32)


for mode in ("tf32x3", "sgemm"):
    if mode == "sgemm":
        F.Fp32StepEngine.gemm = torch_gemm
    for (m, n, b, p) in [(700, 600, 64, 8), (1024, 1000, 128, 16)]:
        a = np.random.default_rng(m).standard_normal((m, n)).astype(np.float32)
        res = F.block_qr_fp32(a, rq.BlockConfig(b, rq.SketchConfig(b, p, 0)), rq.RngState(1), want_q=True)
        a64 = a.astype(np.float64)
        q = res.q.astype(np.float64)
        r = res.r.astype(np.float64)[:n]
        resid = np.linalg.norm(a64[:, res.perm] - q @ r) / np.linalg.norm(a64)
        g = q.T @ q - np.eye(n)
        print(mode, m, n, "resid", resid, "orth2", np.linalg.norm(g, 2), "orthF/sqrt(n)", np.linalg.norm(g) / np.sqrt(n))
