"""Kernel-level parity on the GPU, through the C ABI (librandqr_b200.so).

Checkers: the CPU oracle (oracle/randqr_oracle.py, pinned to the reference in
tests/test_oracle_golden.py) and the golden fixtures of the reference itself.
"""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    from paper_1505_08115_b200 import Engine

    return Engine()


def test_rng_words_bitwise(golden, eng):
    import paper_1505_08115_b200 as rq

    g = golden("rng_kernels.npz")
    assert np.array_equal(rq.splitmix_words(1, 0, 1000, engine=eng), g["rng_words/seed1"])
    assert np.array_equal(rq.splitmix_words(2**63 + 11, 0, 1000, engine=eng), g["rng_words/seed_big"])


def test_rng_normals_match_reference(golden, eng):
    import paper_1505_08115_b200 as rq

    g = golden("rng_kernels.npz")
    for key, val in g.items():
        if not key.startswith("rng/"):
            continue
        _, seed, counter, shape = key.split("/")
        rows, cols = map(int, shape.split("x"))
        rng = rq.RngState(int(seed), int(counter))
        z = rq.gaussian_matrix(rows, cols, rng, engine=eng)
        assert rng.counter == int(counter) + rows * cols
        # integer stream is exact; log/cos differ from numpy's SIMD versions by <= a few ulp
        np.testing.assert_allclose(z, val, rtol=4e-15, atol=4e-15)


def _gemm(eng, a_mmajor, M, N, K, A, B, C, alpha, beta, a_org=(0, 0), b_org=(0, 0)):
    import torch

    def dev(x):
        x = np.asarray(x, dtype=np.float64)
        buf, ld = eng.alloc_matrix(*x.shape)
        buf[: x.shape[1], : x.shape[0]].copy_(torch.from_numpy(np.ascontiguousarray(x.T)))
        return buf, ld

    da, lda = dev(A)
    db, ldb = dev(B)
    dc, ldc = dev(C)
    rc = eng.lib.rq_test_gemm(eng.handle, int(a_mmajor), M, N, K, ctypes.c_void_p(da.data_ptr()), lda,
                              A.shape[0], A.shape[1], a_org[0], a_org[1], ctypes.c_void_p(db.data_ptr()), ldb,
                              B.shape[0], B.shape[1], b_org[0], b_org[1], ctypes.c_void_p(dc.data_ptr()), ldc,
                              alpha, beta)
    from paper_1505_08115_b200.errors import check

    check(rc)
    return eng.download(dc, C.shape[0], C.shape[1])


@pytest.mark.parametrize("M,N,K", [(256, 300, 1000), (16, 8, 4), (130, 37, 45), (272, 2000, 3000), (31, 129, 7),
                                   (1000, 1000, 256)])
@pytest.mark.parametrize("mmajor", [False, True])
def test_dmma_gemm_vs_fp64_reference(eng, M, N, K, mmajor):
    rng = np.random.default_rng(M * 7 + N * 3 + K)
    A = rng.standard_normal((M, K) if mmajor else (K, M))
    B = rng.standard_normal((K, N))
    C = rng.standard_normal((M, N))
    out = _gemm(eng, mmajor, M, N, K, A, B, C, -0.5, 1.5)
    opA = A if mmajor else A.T
    ref = -0.5 * (opA @ B) + 1.5 * C
    tol = 1e-13 * np.sqrt(K) * (np.abs(opA) @ np.abs(B)).max()
    assert np.abs(out - ref).max() <= tol


@pytest.mark.parametrize("M,N,K,org", [(256, 9700, 2100, (0, 0)), (272, 9650, 2049, (1, 3)), (256, 19000, 2064, (0, 0))])
def test_dmma_gemm_whole_waves_plus_split_remainder(eng, M, N, K, org):
    """TN products with a little more than a whole number of tile waves (152 / 152 / 298 tiles on 148
    SMs, K >= 2048) run as whole waves of unsplit tiles plus the remaining tile columns with split-K
    (launch_auto, gemm_f64.cu): same result as one product, also from an offset view."""
    rng = np.random.default_rng(M + N + K)
    r0, c0 = org
    A = rng.standard_normal((K + r0, M + 5))
    B = rng.standard_normal((K + r0, N + c0))
    C = rng.standard_normal((M, N))
    out = _gemm(eng, False, M, N, K, A, B, C, -1.0, 1.0, a_org=(r0, 2), b_org=(r0, c0))
    opA = A[r0:r0 + K, 2:2 + M].T
    Bv = B[r0:r0 + K, c0:c0 + N]
    ref = C - opA @ Bv
    tol = 1e-13 * np.sqrt(K) * (np.abs(opA) @ np.abs(Bv)).max()
    assert np.abs(out - ref).max() <= tol


def test_dmma_gemm_views_and_ktail(eng):
    # views at odd origins, K not a multiple of 16, buffers larger than the views
    rng = np.random.default_rng(5)
    A = rng.standard_normal((90, 70))
    B = rng.standard_normal((90, 50))
    C = rng.standard_normal((33, 21))
    # TN: op(A) = A[3:3+K, 5:5+M]^T, B view rows 3.., cols 7..
    M, N, K = 33, 21, 29
    out = _gemm(eng, False, M, N, K, A, B, C, 1.0, 0.0, a_org=(3, 5), b_org=(3, 7))
    ref = A[3:3 + K, 5:5 + M].T @ B[3:3 + K, 7:7 + N]
    assert np.abs(out - ref).max() <= 1e-12
    # NN: op(A) = A[11:11+M, 2:2+K]
    out = _gemm(eng, True, M, N, K, A, B, C, 1.0, 0.0, a_org=(11, 2), b_org=(3, 7))
    ref = A[11:11 + M, 2:2 + K] @ B[3:3 + K, 7:7 + N]
    assert np.abs(out - ref).max() <= 1e-12


@pytest.mark.parametrize("tag", ["sq", "tall", "wide", "part"])
@pytest.mark.parametrize("pivot", [True, False])
def test_householder_sweep_vs_reference(golden, eng, tag, pivot):
    import paper_1505_08115_b200 as rq
    from oracle import randqr_oracle as O

    g = golden("rng_kernels.npz")
    a0 = g[f"cpqr/{tag}/a"]
    m, n = a0.shape
    steps = min(m, n) if tag != "part" else 32
    if not pivot and m < n:
        steps = min(steps, m)
    a = np.array(a0, order="F")
    v = np.zeros((m, steps), order="F")
    perm = np.arange(n, dtype=np.int64)
    rq.householder_sweep(a, v, perm, steps, pivot, engine=eng)
    ar = np.array(a0, order="F")
    vr = np.zeros((m, steps), order="F")
    pr = np.arange(n, dtype=np.int64)
    O.householder_sweep(ar, vr, pr, steps, pivot)
    if pivot:
        assert np.array_equal(perm, g[f"cpqr/{tag}/perm"])
        assert np.array_equal(perm, pr)
    scale = np.abs(a0).max() * max(m, n)
    assert np.abs(a - ar).max() <= 1e-13 * scale
    assert np.abs(v - vr).max() <= 1e-12
    assert np.array_equal(np.sign(np.diag(a)), np.sign(np.diag(ar)))


def test_householder_sweep_ties_lowest_index(golden, eng):
    import paper_1505_08115_b200 as rq

    g = golden("rng_kernels.npz")
    a = np.array(g["cpqr/ties/a"], order="F")
    m, n = a.shape
    v = np.zeros((m, min(m, n)), order="F")
    perm = np.arange(n, dtype=np.int64)
    rq.householder_sweep(a, v, perm, min(m, n), True, engine=eng)
    # the genuine tie (columns 1 and 3, equal norms) goes to the lowest index
    assert perm[0] == g["cpqr/ties/perm"][0] == 1
    # afterwards every trailing column is zero up to rounding: any order is a valid CPQR
    assert np.abs(np.diag(a)[1:]).max() <= 1e-15


def test_hand_examples(eng):
    # pkg/tests/test_householder.py:114-131 and :163-173
    import paper_1505_08115_b200 as rq

    a = np.array([[3.0, 0.0], [4.0, 5.0]], order="F")
    v = np.zeros((2, 2), order="F")
    rq.householder_sweep(a, v, np.arange(2), 2, False, engine=eng)
    assert np.abs(a - [[-5.0, -4.0], [0.0, 3.0]]).max() <= 1e-13
    a = np.array([[0.0, 2.0], [0.0, 1.0]], order="F")
    perm = np.arange(2, dtype=np.int64)
    rq.householder_sweep(a, np.zeros((2, 2), order="F"), perm, 2, True, engine=eng)
    assert perm.tolist() == [1, 0]
    assert abs(a[0, 0]) == pytest.approx(np.sqrt(5.0), abs=1e-14)
    a = np.eye(4, order="F")
    perm = np.arange(4, dtype=np.int64)
    rq.householder_sweep(a, np.zeros((4, 4), order="F"), perm, 4, True, engine=eng)
    assert perm.tolist() == [0, 1, 2, 3]


@pytest.mark.parametrize("m,n,steps", [(74, 2000, 64), (272, 1000, 256), (272, 10000, 256), (272, 20000, 256),
                                       (272, 30000, 256), (272, 40000, 256)])
def test_sketch_cpqr_tiers_choose_the_oracle_pivots(eng, m, n, steps):
    """The sketch CPQR's register tier (n' <= 11.8k at b + p = 272), shared-memory tier (<= 23k) and
    L2-resident tier (<= 53k) pick the oracle's CPQR pivots (pivoting.py:114-129 via
    householder_sweep), and leave Y untouched."""
    import torch

    from oracle import randqr_oracle as O
    from paper_1505_08115_b200.errors import check

    y = np.random.default_rng(m + n).standard_normal((m, n))
    buf, ld = eng.alloc_matrix(m, n)
    buf[:n, :m].copy_(torch.from_numpy(np.ascontiguousarray(y.T)))
    before = buf.clone()
    ch = torch.zeros(steps, dtype=torch.int32, device=eng.device)
    check(eng.lib.rq_test_sketch_cpqr(eng.handle, ctypes.c_void_p(buf.data_ptr()), ld, m, n, steps,
                                      ctypes.c_void_p(ch.data_ptr())))
    torch.cuda.synchronize()
    ref = O.qr_column_pivoted(y, steps=steps).perm[:steps]
    assert np.array_equal(ch.cpu().numpy().astype(np.int64), ref)
    assert torch.equal(buf, before)


def test_exchange_kernels_repeatable_under_stress():
    """compute-sanitizer is closed on this pool (profiles/sanitizer_r02_closed.txt), so the
    fence-free exchanges (LL-stamped grid words of sketch_reg_kernel, st.async cluster pushes of
    sweep_reg_kernel / leaf_reg_kernel) are stress-tested instead: many back-to-back launches on
    fresh inputs, every result bitwise equal to a first run and the pivots to the oracle's."""
    import ctypes

    import torch

    import paper_1505_08115_b200 as rq
    from oracle import randqr_oracle as O
    from paper_1505_08115_b200.errors import check

    eng = rq.Engine()
    lib = eng.lib
    rng = np.random.default_rng(123)

    def dev(x):
        buf, ld = eng.alloc_matrix(*x.shape)
        buf[: x.shape[1], : x.shape[0]].copy_(torch.from_numpy(np.ascontiguousarray(x.T)))
        return buf, ld

    for (m, n, steps) in [(272, 3000, 256), (74, 1200, 64), (272, 9000, 128)]:
        y0 = rng.standard_normal((m, n))
        src, ld = dev(y0)
        work, _ = eng.alloc_matrix(m, n)
        outs = []
        for _ in range(40):
            work.copy_(src)
            ch = torch.zeros(steps, dtype=torch.int32, device=eng.device)
            check(lib.rq_test_sketch_cpqr(eng.handle, ctypes.c_void_p(work.data_ptr()), ld, m, n, steps,
                                          ctypes.c_void_p(ch.data_ptr())))
            outs.append(ch)
        ref = outs[0].cpu().numpy()
        for o in outs[1:]:
            assert np.array_equal(o.cpu().numpy(), ref)
        assert np.array_equal(ref.astype(np.int64), O.qr_column_pivoted(y0, steps=steps).perm[:steps]), (m, n)
    for k in (96, 256):
        a0 = rng.standard_normal((k, k))
        src, ld = dev(a0)
        work, _ = eng.alloc_matrix(k, k)
        v, ldv = eng.alloc_matrix(k, k)
        first = None
        for _ in range(60):
            work.copy_(src)
            v.zero_()
            perm = torch.arange(k, dtype=torch.int64, device=eng.device)
            check(lib.rq_householder_sweep(eng.handle, ctypes.c_void_p(work.data_ptr()), k, k, ld,
                                           ctypes.c_void_p(v.data_ptr()), ldv, ctypes.c_void_p(perm.data_ptr()), k, 1))
            got = (perm.cpu().numpy(), work[:k, :k].cpu().numpy().copy())
            if first is None:
                first = got
            else:
                assert np.array_equal(got[0], first[0]) and np.array_equal(got[1], first[1])
        assert np.array_equal(first[0], O.qr_column_pivoted(a0).perm)
    for (mm, w) in [(3000, 16), (700, 32)]:
        a0 = rng.standard_normal((mm, w))
        src, ld = dev(a0)
        work, _ = eng.alloc_matrix(mm, w)
        v, ldv = eng.alloc_matrix(mm, w)
        t, ldt = eng.alloc_matrix(32, 32)
        first = None
        for _ in range(60):
            work.copy_(src)
            check(lib.rq_test_leaf_qr(eng.handle, ctypes.c_void_p(work.data_ptr()), ld, mm, w,
                                      ctypes.c_void_p(v.data_ptr()), ldv, ctypes.c_void_p(t.data_ptr()), ldt))
            got = work[:w, :mm].cpu().numpy().copy()
            if first is None:
                first = got
            else:
                assert np.array_equal(got, first)
        r_ref = O.qr_unpivoted(a0).r[:w, :]
        assert np.abs(np.triu(first.T[:w, :]) - r_ref).max() <= 1e-12 * np.linalg.norm(a0)


def test_batched_sketch_cpqr_opt_in_picks_the_same_pivots():
    """RQ_SK_BATCH=1 (sketch_batch.cu: one grid exchange per provable batch of pivots, opt-in because it
    measured at parity with the per-step kernel) returns the per-step kernel's pivots bit for bit -- also
    on duplicated columns, zero columns and beyond the numerical rank -- and the oracle's where those are
    well determined.  The switch is read once per process, hence the subprocess."""
    import os
    import subprocess
    import sys

    code = r"""
import ctypes, sys
import numpy as np, torch
import paper_1505_08115_b200 as rq
from paper_1505_08115_b200.errors import check
eng = rq.Engine()
rng = np.random.default_rng(11)
cases = []
cases.append(("gauss", rng.standard_normal((272, 3000)), 256))
y = rng.standard_normal((272, 3000)); y[:, 100] = y[:, 2500]; y[:, 1500:1510] = y[:, 20:21]
cases.append(("dups", y, 256))
cases.append(("rank40", rng.standard_normal((272, 40)) @ rng.standard_normal((40, 2500)), 100))
y = rng.standard_normal((80, 500)); y[:, 50:] = 0.0
cases.append(("zeros", y, 70))
cases.append(("small", rng.standard_normal((74, 1200)), 64))
cases.append(("wide", rng.standard_normal((272, 14000)), 128))
out = {}
for name, y, steps in cases:
    m, n = y.shape
    buf, ld = eng.alloc_matrix(m, n)
    buf[:n, :m].copy_(torch.from_numpy(np.ascontiguousarray(y.T)))
    before = buf.clone()
    ch = torch.full((steps,), -1, dtype=torch.int32, device=eng.device)
    check(eng.lib.rq_test_sketch_cpqr(eng.handle, ctypes.c_void_p(buf.data_ptr()), ld, m, n, steps,
                                      ctypes.c_void_p(ch.data_ptr())))
    torch.cuda.synchronize()
    assert torch.equal(buf, before), name
    out[name] = ch.cpu().numpy()
np.savez(sys.argv[1], **out)
"""
    import tempfile

    from oracle import randqr_oracle as O

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    with tempfile.TemporaryDirectory() as d:
        for flag in ("0", "1"):
            path = os.path.join(d, f"p{flag}.npz")
            env = dict(os.environ, RQ_SK_BATCH=flag, PYTHONPATH=root)
            r = subprocess.run([sys.executable, "-c", code, path], env=env, capture_output=True, text=True, timeout=600)
            assert r.returncode == 0, r.stderr[-2000:]
            res[flag] = dict(np.load(path))
    for name in res["0"]:
        assert np.array_equal(res["0"][name], res["1"][name]), name
    rng = np.random.default_rng(11)
    y = rng.standard_normal((272, 3000))
    assert np.array_equal(res["1"]["gauss"].astype(np.int64), O.qr_column_pivoted(y, steps=256).perm[:256])


@pytest.mark.parametrize("reducer", ["0", "1", "2"])
def test_sketch_cpqr_placement_calibration_with_every_reducer_mode(reducer):
    """The one-off placement calibration of the sketch CPQR's exchange words (driver.cu place_sketch_words,
    triggered by the first sketch with >= 2048 columns) runs the kernel on 16 candidate records: with the
    arrival-counter reducer (RQ_SK_FIXED_REDUCER=0) every candidate's device counter must match the host
    mirror or the launch never ends -- run each mode in a subprocess under a timeout and check the pivots."""
    import os
    import subprocess
    import sys

    code = r"""
import ctypes, sys
import numpy as np, torch
import paper_1505_08115_b200 as rq
from oracle import randqr_oracle as O
from paper_1505_08115_b200.errors import check
eng = rq.Engine()
rng = np.random.default_rng(3)
for (m, n, steps) in [(272, 2600, 128), (272, 900, 64), (74, 2100, 48)]:
    y = rng.standard_normal((m, n))
    buf, ld = eng.alloc_matrix(m, n)
    buf[:n, :m].copy_(torch.from_numpy(np.ascontiguousarray(y.T)))
    ch = torch.full((steps,), -1, dtype=torch.int32, device=eng.device)
    for _ in range(2):
        check(eng.lib.rq_test_sketch_cpqr(eng.handle, ctypes.c_void_p(buf.data_ptr()), ld, m, n, steps,
                                          ctypes.c_void_p(ch.data_ptr())))
        torch.cuda.synchronize()
        assert np.array_equal(ch.cpu().numpy().astype(np.int64), O.qr_column_pivoted(y, steps=steps).perm[:steps])
print("OK")
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, RQ_SK_FIXED_REDUCER=reducer, PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=180)
    assert r.returncode == 0 and "OK" in r.stdout, r.stderr[-2000:]
