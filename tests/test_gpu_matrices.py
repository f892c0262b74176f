"""Device-side test matrices and metrics vs the reference
algorithm: unpivoted QR (householder.py:152-161), haar_orthonormal / gen_matrix
(matrices.py:34-71), Frobenius truncation errors (metrics.py:37-52)."""

import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "oracle"))

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,n,block", [(300, 300, 64), (517, 333, 128), (1000, 1000, 256)])
def test_qr_unpivoted_matches_reference(m, n, block):
    import ctypes

    import randqr_oracle as orc
    import paper_1505_08115_b200 as rq

    a = np.random.default_rng(m + n).standard_normal((m, n))
    eng = rq.Engine()
    buf, ld, _, _ = eng.upload(a)
    assert eng.lib.rq_qr_unpivoted(eng.handle, m, n, ctypes.c_void_p(buf.data_ptr()), ld, block) == 0
    r = rq.Engine.download(buf, m, n)
    ref = orc.qr_unpivoted(a)
    assert np.abs(np.triu(r) - ref.r).max() <= 1e-13 * np.linalg.norm(a)
    q, ldq = eng.alloc_matrix(m, n)
    assert eng.lib.rq_form_q(eng.handle, n, ctypes.c_void_p(q.data_ptr()), ldq) == 0
    qm = rq.Engine.download(q, m, n)
    assert np.linalg.norm(qm @ np.triu(r)[:n] - a) <= 1e-13 * np.linalg.norm(a)


def test_haar_orthonormal_matches_reference():
    import randqr_oracle as orc
    from paper_1505_08115_b200 import RngState
    from paper_1505_08115_b200.matrices import haar_orthonormal

    n = 400
    rng, ref_rng = RngState(0), orc.RngState(0)
    q = haar_orthonormal(n, rng)
    q_ref = orc.haar_orthonormal(n, ref_rng)
    assert np.abs(q - q_ref).max() <= 1e-12
    assert rng.counter == ref_rng.counter == n * n


@pytest.mark.parametrize("kind", ["fast", "sshape"])
def test_gen_matrix_matches_reference_construction(kind):
    import randqr_oracle as orc
    from paper_1505_08115_b200.matrices import MatrixSpec, _sigma, gen_matrix

    n, seed = 300, 4
    a, d = gen_matrix(MatrixSpec(kind, n, seed))
    rr = orc.RngState(seed)
    u = orc.haar_orthonormal(n, rr)
    v = orc.haar_orthonormal(n, rr)  # U is drawn before V (matrices.py:67-68)
    a_ref = (u * _sigma(kind, n)) @ v.T
    assert np.abs(a - a_ref).max() <= 1e-12
    assert np.array_equal(d, _sigma(kind, n))


def test_truncation_errors_frobenius_vs_dense():
    import paper_1505_08115_b200 as rq
    from paper_1505_08115_b200.matrices import MatrixSpec, gen_matrix, truncation_errors_frobenius

    n, b = 256, 32
    a, _ = gen_matrix(MatrixSpec("fast", n, 1))
    f = rq.block_qr(a, rq.BlockConfig(b, rq.SketchConfig(b, 8, 0)), rq.RngState(2))
    ks = list(range(0, n, b)) + [n]
    got = truncation_errors_frobenius(f, ks)
    q, p = f.expand_q(), f.expand_p()
    rp = f.r[:n, :] @ p.T
    for k, e in zip(ks, got):
        dense = np.linalg.norm(a - q[:, :k] @ rp[:k, :]) if k > 0 else np.linalg.norm(a)
        assert abs(e - dense) <= 1e-12 * np.linalg.norm(a) + 1e-10 * dense


def test_truncation_errors_spectral_and_frobenius_match_dense():
    """metrics.truncation_errors (metrics.py:37-52) from R on the device -- Jacobi SVD kernel for
    trailing blocks <= 512 wide, power iteration beyond -- against the dense definition."""
    import paper_1505_08115_b200 as rq
    from paper_1505_08115_b200 import metrics

    rng = np.random.default_rng(4)
    n = 700
    s = 10.0 ** (-3.0 * np.arange(n) / n)
    u, _ = np.linalg.qr(rng.standard_normal((n, n)))
    v, _ = np.linalg.qr(rng.standard_normal((n, n)))
    a = np.asfortranarray((u * s) @ v.T)
    f = rq.block_qr(a, rq.BlockConfig(64, rq.SketchConfig(64, 8, 0)), rq.RngState(1))
    ks = [0, 64, 150, 188, 600, 700]
    c = metrics.truncation_errors(a, f, ks)
    q, p = f.expand_q(), f.expand_p()
    rp = f.r[:n, :] @ p.T
    for i, k in enumerate(ks):
        resid = a - q[:, :k] @ rp[:k, :] if k else a
        fro = np.linalg.norm(resid)
        sp = np.linalg.norm(resid, 2) if k < n else 0.0
        assert abs(c.frobenius[i] - fro) <= 1e-12 * np.linalg.norm(a), (k, c.frobenius[i], fro)
        tol = 1e-9 if n - k > 512 else 1e-12
        assert abs(c.spectral[i] - sp) <= tol * max(sp, 1e-300) + 1e-13 * np.linalg.norm(a), (k, c.spectral[i], sp)
    d = metrics.diag_comparison(f, s)
    assert np.array_equal(d.r_abs, np.abs(np.diag(f.r)))
