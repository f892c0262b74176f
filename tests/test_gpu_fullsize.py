"""Full-size parity on the BASELINE configs against fixtures the REFERENCE produced
(tests/golden/make_golden_large.py runs randqr.block_qr / block_rrqr in the build container).

The GPU regenerates each input on the device with the same streams (rng.py:54-68,
matrices.py:34-41); the normals agree with numpy's to ~1 ulp, so the
fixture's checksums of A are compared to a tight relative tolerance first.

Bars (north_star, SURVEY section 8c "diag(R) parity caveat"):
  * identical composite permutation (all n entries) and RNG counter;
  * identical signs of diag(R);
  * |R_jj - R_jj,ref| <= 1e-10 |R_jj,ref| where |R_jj,ref| >= 1e-6 ||A||_F,
    and <= 1e-14 ||A||_F everywhere.
"""

import ctypes
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _fixture(name):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not generated (tests/golden/make_golden_large.py)")
    return dict(np.load(path))


@pytest.fixture(scope="module")
def rq():
    import paper_1505_08115_b200 as m

    return m


def _checksum_close(a_dev_t, ref):
    """a_dev_t: torch (n x n) view of A on the device."""
    import torch

    got = np.array([float(a_dev_t.sum()), float(a_dev_t.abs().sum()), float(a_dev_t[0, 0]), float(a_dev_t[-1, -1]),
                    float(torch.linalg.norm(a_dev_t[:, 0]))])
    assert np.all(np.abs(got - ref) <= 1e-9 * np.maximum(np.abs(ref), 1.0)), (got, ref)


def _factorize_device(rq, eng, a_store, ld, m, n, b, p, q=0, mode=0, refl=False, rr=False, seed=1):
    import torch

    from paper_1505_08115_b200 import _lib
    from paper_1505_08115_b200.errors import check

    work = a_store.clone()
    perm = torch.empty(n, dtype=torch.int64, device=a_store.device)
    pk = _lib.RQ_PIVOT_REFLECTORS if (refl or rr) else _lib.RQ_PIVOT_PERMUTATION
    cfg = _lib.rq_config(b, p, q, -1, pk, int(rr), mode, 0)
    ctr = ctypes.c_uint64(0)
    check(eng.lib.rq_factorize(eng.handle, ctypes.byref(cfg), m, n, ctypes.c_void_p(work.data_ptr()), ld,
                               ctypes.c_uint64(seed), ctypes.byref(ctr),
                               None if (refl or rr) else ctypes.c_void_p(perm.data_ptr())))
    return work, perm, ctr.value


def _diag_parity(d, dref, anorm):
    assert np.array_equal(np.sign(d), np.sign(dref))
    big = np.abs(dref) >= 1e-6 * anorm
    assert np.all(np.abs(d[big] - dref[big]) <= 1e-10 * np.abs(dref[big]))
    assert np.abs(d - dref).max() <= 1e-14 * anorm


def test_cfg3_n10k_full_permutation_and_diag_match_reference(rq):
    """BASELINE cfg 3 (fp64): A = gaussian_matrix(10000, 10000, RngState(0)), b = 256, p = 16,
    fresh sketches from RngState(1) -- the reference's own block_qr run (blocked.py:175-219,
    ~150-300 s on the CPU) pinned all 10 000 pivots and diag(R)."""
    import torch

    g = _fixture("cfg3_n10000.npz")
    n, b, p = 10000, 256, 16
    eng = rq.Engine()
    a, ld = rq.gaussian_matrix_device(n, n, rq.RngState(0), engine=eng)
    _checksum_close(a[:n, :n].T, g["a_checksum"])
    work, perm, ctr = _factorize_device(rq, eng, a, ld, n, n, b, p)
    assert ctr == int(g["counter"])
    got = perm.cpu().numpy()
    ref = g["perm"].astype(np.int64)
    assert np.array_equal(got, ref), f"first mismatch at {int(np.argmax(got != ref))}"
    d = torch.diagonal(work[:n, :n]).cpu().numpy()
    anorm = float(torch.linalg.norm(a[:n, :n]))
    _diag_parity(d, g["diag"], anorm)
    rtop = work[:n, :8].T.cpu().numpy()  # rows 0..7 of R
    assert np.abs(rtop - g["r_top"]).max() <= 1e-13 * anorm


def _haar_matrix(rq, eng, n, s):
    import torch

    from paper_1505_08115_b200.matrices import haar_orthonormal_device

    hr = rq.RngState(0)
    u, _ = haar_orthonormal_device(n, hr, engine=eng)
    v, _ = haar_orthonormal_device(n, hr, engine=eng)
    st = torch.as_tensor(s, device=u.device)
    a, ld = eng.alloc_matrix(n, n)
    a[:n, :n] = v[:n, :n].T @ (u[:n, :n] * st[:, None])  # storage(A) = A^T = V diag(s) U^T
    return a, ld


def test_cfg2_n4000_permutation_and_diag_match_reference(rq):
    """BASELINE cfg 2: A = U diag(10^(-8 j/n)) V^T, n = 4000, U, V = haar_orthonormal(4000,
    RngState(0)) built on the device; block_qr b = 128, p = 10, RngState(1), vs the reference."""
    import torch

    g = _fixture("cfg2_n4000.npz")
    n, b, p = 4000, 128, 10
    eng = rq.Engine()
    a, ld = _haar_matrix(rq, eng, n, g["s"])
    at = a[:n, :n].T
    assert abs(float(at.abs().sum()) - g["a_checksum"][1]) <= 1e-9 * g["a_checksum"][1]
    work, perm, ctr = _factorize_device(rq, eng, a, ld, n, n, b, p)
    assert ctr == int(g["counter"])
    got = perm.cpu().numpy()
    ref = g["perm"].astype(np.int64)
    assert np.array_equal(got, ref), f"first mismatch at {int(np.argmax(got != ref))}"
    d = torch.diagonal(work[:n, :n]).cpu().numpy()
    _diag_parity(d, g["diag"], float(torch.linalg.norm(at)))


def test_cfg4_n8000_rrqr_diag_tracks_reference(rq):
    """BASELINE cfg 4: block_rrqr (blocked.py:239-279), n = 8000, b = 128, p = 10, q = 1,
    A = U diag(max(10^(-12 j/2000), 1e-15)) V^T.  The reference reached max_{j<2000}
    |R_jj/s_j - 1| = 0.276; the B200 run must agree with the reference's
    diag(R) where the q = 1 sketch determines it (|R_jj| >= 1e-2 ||A||, see
    test_gpu_block_qr.test_block_rrqr_cfg4_like_spectrum) and stay in the same quality class."""
    import torch

    g = _fixture("cfg4_n8000.npz")
    n, b, p, q = 8000, 128, 10, 1
    s = g["s"]
    eng = rq.Engine()
    a, ld = _haar_matrix(rq, eng, n, s)
    at = a[:n, :n].T
    assert abs(float(at.abs().sum()) - g["a_checksum"][1]) <= 1e-9 * g["a_checksum"][1]
    work, _, ctr = _factorize_device(rq, eng, a, ld, n, n, b, p, q=q, rr=True)
    assert ctr == int(g["counter"])
    d = torch.diagonal(work[:n, :n]).cpu().numpy()
    ref = g["diag"]
    anorm = float(torch.linalg.norm(at))
    big = ref >= 1e-2 * anorm
    assert big.sum() >= 100
    assert np.all(np.abs(d[big] - ref[big]) <= 1e-10 * ref[big])
    dev = np.abs(d[:2000] / s[:2000] - 1.0)
    dev_ref = np.abs(ref[:2000] / s[:2000] - 1.0)
    assert dev.max() <= dev_ref.max() + 0.1, (dev.max(), dev_ref.max())
    assert np.median(dev) <= np.median(dev_ref) + 0.01
    # diagonal blocks exactly diagonal, >= 0, non-increasing (pkg/tests/test_blocked.py:128-139)
    r = work[:n, :n].T
    for s0 in range(0, n, b):
        blk = r[s0:s0 + b, s0:s0 + b]
        dd = torch.diagonal(blk)
        assert torch.equal(blk, torch.diag(dd))
        assert bool((dd >= 0).all()) and bool((dd[1:] <= dd[:-1]).all())


def test_downdate_n10k_permutation_matches_post_rotation_oracle(rq):
    """The headline mode (HQRRP downdated sketch, look-ahead schedule) at the bench size, against
    the oracle's independent post-rotation restatement (block_qr_downdate(form="post")) run on the
    reference's A: all 10 000 pivots identical, diag(R) to the bars above."""
    import torch

    g = _fixture("downdate_n10000.npz")
    n, b, p = 10000, 256, 16
    eng = rq.Engine()
    a, ld = rq.gaussian_matrix_device(n, n, rq.RngState(0), engine=eng)
    _checksum_close(a[:n, :n].T, g["a_checksum"])
    work, perm, ctr = _factorize_device(rq, eng, a, ld, n, n, b, p, mode=1)
    assert ctr == int(g["counter"]) == n * (b + p)
    got = perm.cpu().numpy()
    ref = g["perm"].astype(np.int64)
    assert np.array_equal(got, ref), f"first mismatch at {int(np.argmax(got != ref))}"
    d = torch.diagonal(work[:n, :n]).cpu().numpy()
    _diag_parity(d, g["diag"], float(torch.linalg.norm(a[:n, :n])))
