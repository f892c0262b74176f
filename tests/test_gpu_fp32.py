"""fp32 path (paper_1505_08115_b200/fp32.py): fp32 storage, the sketch / trailing update / Q
formation on this library's tcgen05 3xTF32 GEMM, fp64 serial kernels.  No reference exists in fp32
(the reference is fp64-only); judged by the north star's fp32 bars -- ||AP - QR||_F / ||A||_F <=
1e-5 and ||Q^T Q - I|| <= 1e-5 (spectral; Frobenius normalised by sqrt(n) as the reference's own
tests do, test_blocked.py:29) -- and by its pivots against the fp64 path on a well-separated
spectrum."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _bars(a, res):
    a64 = a.astype(np.float64)
    q = res.q.astype(np.float64)
    r = res.r.astype(np.float64)[: a.shape[1]]
    n = a.shape[1]
    resid = np.linalg.norm(a64[:, res.perm] - q @ r) / np.linalg.norm(a64)
    g = q.T @ q - np.eye(n)
    return resid, np.linalg.norm(g, 2), np.linalg.norm(g) / np.sqrt(n)


@pytest.mark.parametrize("m,n,b,p,sketch", [(700, 600, 64, 8, "fresh"), (1024, 1000, 128, 16, "fresh"),
                                            (530, 500, 50, 6, "fresh"), (1024, 1000, 128, 16, "downdate"),
                                            (530, 500, 50, 6, "downdate")])
def test_fp32_q_based_residuals_and_counter(m, n, b, p, sketch):
    import paper_1505_08115_b200 as rq
    from paper_1505_08115_b200.fp32 import block_qr_fp32

    a = np.random.default_rng(m).standard_normal((m, n)).astype(np.float32)
    cfg = rq.BlockConfig(b, rq.SketchConfig(b, p, 0))
    rng32, rng64 = rq.RngState(1), rq.RngState(1)
    res = block_qr_fp32(a, cfg, rng32, want_q=True, sketch=sketch, driver="steps")
    f = rq.block_qr(a.astype(np.float64), cfg, rng64, sketch=sketch)
    assert res.r.dtype == np.float32 and res.q.dtype == np.float32
    assert sorted(res.perm) == list(range(n))
    resid, orth2, orthf = _bars(a, res)
    assert resid <= 1e-5, resid
    assert orth2 <= 1e-5, orth2
    assert orthf <= 1e-5, orthf
    assert not np.tril(res.r, -1).any()
    assert rng32.counter == rng64.counter
    assert np.mean(res.perm == f.perm) > 0.5


def test_fp32_bench_size_n10k_residual_probes():
    """cfg 3 fp32 at its full size (n = 10000, b = 256, p = 16): the fp32 bars through random
    probes on the device (||A[:, perm] x - Q (R x)|| / (||A|| ||x||), ||Q^T Q y - y|| / ||y||)."""
    import torch

    import paper_1505_08115_b200 as rq
    from paper_1505_08115_b200 import dist as rqd
    from paper_1505_08115_b200.fp32 import Fp32StepEngine

    n, b, p = 10000, 256, 16
    eng = rq.Engine()
    se = Fp32StepEngine(eng, keep_factors=True)
    a64, _ = rq.gaussian_matrix_device(n, n, rq.RngState(0), engine=eng)
    a0, lda = se.alloc(n, n)
    a0[:n, :n] = a64[:n, :n]
    del a64
    work = a0.clone()
    res = rqd.factorize_local(work, lda, n, n, rq.BlockConfig(b, rq.SketchConfig(b, p, 0)), rq.RngState(1),
                              engine=se)
    q, _ = se.form_q(n, n)
    A = a0[:n, :n].T.double()
    R = torch.triu(work[:n, :n].T.double())
    Q = q[:n, :n].T.double()
    perm = torch.as_tensor(res.perm, device=A.device)
    g = torch.Generator(device=A.device).manual_seed(3)
    x = torch.randn(n, 4, dtype=torch.float64, device=A.device, generator=g)
    r1 = torch.linalg.norm(A[:, perm] @ x - Q @ (R @ x)) / (torch.linalg.norm(A) * torch.linalg.norm(x))
    assert float(r1) <= 1e-5, float(r1)
    y = torch.randn(n, 4, dtype=torch.float64, device=A.device, generator=g)
    r2 = torch.linalg.norm(Q.T @ (Q @ y) - y) / torch.linalg.norm(y)
    assert float(r2) <= 1e-5, float(r2)


def test_fp32_leading_pivots_on_graded_spectrum():
    import paper_1505_08115_b200 as rq
    from paper_1505_08115_b200.fp32 import block_qr_fp32

    n, b, p = 512, 64, 8
    rng = np.random.default_rng(3)
    u, _ = np.linalg.qr(rng.standard_normal((n, n)))
    v, _ = np.linalg.qr(rng.standard_normal((n, n)))
    s = 0.93 ** np.arange(n)  # well-separated down to ~1e-16: compare where fp32 resolves it
    a64 = (u * s) @ v.T
    cfg = rq.BlockConfig(b, rq.SketchConfig(b, p, 0))
    res = block_qr_fp32(a64.astype(np.float32), cfg, rq.RngState(1), driver="steps")
    mono = block_qr_fp32(a64.astype(np.float32), cfg, rq.RngState(1))  # the monolithic tf32-update driver
    f = rq.block_qr(a64, cfg, rq.RngState(1))
    k = 96  # s_k ~ 1e-3: sketch norms far above fp32 rounding
    assert np.array_equal(res.perm[:k], f.perm[:k])
    assert np.array_equal(mono.perm[:k], f.perm[:k])
    d32, d64 = np.abs(np.diag(res.r))[:k], np.abs(np.diag(f.r))[:k]
    assert np.all(np.abs(d32 - d64) <= 1e-4 * d64 + 1e-6)


@pytest.mark.parametrize("m,n,b,p,sketch", [(700, 600, 64, 8, "fresh"), (1024, 1000, 128, 16, "downdate"),
                                            (530, 500, 50, 6, "downdate"), (3000, 3000, 256, 16, "downdate")])
def test_tf32_update_mode_fp32_bars(m, n, b, p, sketch):
    """The monolithic driver's fp32 path (RQ_FLAG_TF32_UPDATE: trailing-update GEMMs as 3xTF32
    tcgen05 products, fp64 panels): Q-based bars at the north star's fp32 level (1e-5), the same
    RNG counter as fp64, and pivots equal to fp64's on the leading panel."""
    import paper_1505_08115_b200 as rq

    a = np.random.default_rng(m + 1).standard_normal((m, n))
    cfg = rq.BlockConfig(b, rq.SketchConfig(b, p, 0))
    r1, r2 = rq.RngState(1), rq.RngState(1)
    f = rq.block_qr(a, cfg, r1, sketch=sketch, tf32_update=True)
    f64 = rq.block_qr(a, cfg, r2, sketch=sketch)
    assert r1.counter == r2.counter
    q = f.expand_q()
    resid = np.linalg.norm(a[:, f.perm] - q @ f.r[:n]) / np.linalg.norm(a)
    orth = np.linalg.norm(q.T @ q - np.eye(n), 2)
    assert resid <= 1e-5 and orth <= 1e-5, (resid, orth)
    assert resid >= 1e-9  # the update really ran at fp32 accuracy (fp64 gives ~1e-15)
    assert np.array_equal(f.perm[:b], f64.perm[:b])
    assert not np.tril(f.r, -1).any()
