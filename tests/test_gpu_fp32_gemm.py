"""The fp32 path's own GEMM (rq_gemm_f32: 3xTF32 split products on tcgen05 tensor cores, TMA
staging, TMEM accumulator) against an fp64 numpy product of the same fp32 inputs.  Bar: fp32
accuracy, |C - C_ref| <= 4e-6 * sum_k |A_ik| |B_kj| (a plain TF32 product misses it by ~100x)."""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    import paper_1505_08115_b200 as rq

    return rq.Engine()


def _buf(torch, eng, rows, cols, rng):
    ld = (rows + 3) // 4 * 4 + 4
    t = torch.from_numpy(rng.standard_normal((cols, ld)).astype(np.float32)).to(eng.device)
    return t, ld


@pytest.mark.parametrize("mmajor,M,N,K,r0a,c0a,r0b,c0b,alpha,beta", [
    (0, 256, 700, 1000, 0, 0, 0, 0, 1.0, 0.0),      # W = V^T A2 (TN)
    (0, 272, 333, 517, 8, 3, 8, 5, 1.0, 0.0),       # sketch-like M = b + p, K / origin tails
    (1, 900, 500, 256, 0, 0, 0, 0, -1.0, 1.0),      # A2 -= V W2 (NN)
    (1, 130, 257, 64, 6, 2, 12, 1, 0.5, -2.0),      # unaligned M origin of an M-major A
    (0, 128, 128, 32, 0, 0, 0, 0, 1.0, 1.0),
    (0, 64, 40, 7, 2, 0, 2, 0, 1.0, 0.0),           # one partial tile, K < 8
    (1, 1000, 1300, 1000, 4, 0, 0, 4, 1.0, 0.0),    # square-ish, many k-blocks
])
def test_gemm_f32_matches_fp64_product(eng, mmajor, M, N, K, r0a, c0a, r0b, c0b, alpha, beta):
    import torch

    from paper_1505_08115_b200.errors import check

    rng = np.random.default_rng(M * 7 + N + K)
    a_rows, a_cols = (M + r0a, K + c0a) if mmajor else (K + r0a, M + c0a)
    a, lda = _buf(torch, eng, a_rows, a_cols, rng)
    b, ldb = _buf(torch, eng, K + r0b, N + c0b, rng)
    c, ldc = _buf(torch, eng, M, N, rng)
    A = a.cpu().numpy().astype(np.float64)[:a_cols, :a_rows].T  # (rows, cols) column-major view
    Bm = b.cpu().numpy().astype(np.float64)[:N + c0b, :K + r0b].T
    C0 = c.cpu().numpy().astype(np.float64)[:N, :M].T
    opa = A[r0a:r0a + M, c0a:c0a + K] if mmajor else A[r0a:r0a + K, c0a:c0a + M].T
    bb = Bm[r0b:r0b + K, c0b:c0b + N]
    ref = alpha * opa @ bb + beta * C0
    check(eng.lib.rq_gemm_f32(eng.handle, mmajor, M, N, K, ctypes.c_void_p(a.data_ptr()), lda, a_rows, a_cols, r0a,
                              c0a, ctypes.c_void_p(b.data_ptr()), ldb, K + r0b, N + c0b, r0b, c0b,
                              ctypes.c_void_p(c.data_ptr()), ldc, alpha, beta))
    got = c.cpu().numpy().astype(np.float64)[:N, :M].T
    scale = abs(alpha) * np.abs(opa) @ np.abs(bb) + abs(beta) * np.abs(C0)
    err = np.abs(got - ref) / np.maximum(scale, 1e-30)
    assert err.max() <= 4e-6, err.max()
    # untouched memory around the output (rows of the padded leading dimension)
    full = c.cpu().numpy()
    assert np.isfinite(full).all()
