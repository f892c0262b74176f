"""GPU tests of the panel-step C ABI and of the multi-GPU driver's CUDA engine.

* rq_panel_factor / rq_panel_apply / rq_sketch_select against the oracle's
  qr_tall_pivoted (householder.py:183-198), trailing update
  (householder.py:105-114) and select_pivot_permutation (pivoting.py:114-129);
* dist.block_qr_distributed over a world-size-1 NCCL group, CUDA step engine, against
  the monolithic GPU driver and the oracle (identical permutation, R to 1e-12 ||A||).
  Ranks > 1 are covered on CPU by tests/test_dist.py (gloo).
"""

import os
import socket
import sys

import numpy as np
import pytest

_HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(_HERE, ".."))
sys.path.insert(0, os.path.join(_HERE, "..", "oracle"))

pytestmark = pytest.mark.gpu


def _eng():
    from paper_1505_08115_b200.dist import CudaStepEngine

    return CudaStepEngine()


def _put(buf, x):
    import torch

    buf[:x.shape[1], :x.shape[0]].copy_(torch.from_numpy(np.ascontiguousarray(x.T)))


def _get(buf, rows, cols):
    return np.asfortranarray(buf[:cols, :rows].cpu().numpy().T)


@pytest.mark.parametrize("mp,b", [(700, 64), (333, 50), (2000, 256)])
def test_panel_factor_matches_oracle(mp, b):
    import randqr_oracle as orc

    e = _eng()
    a = np.random.default_rng(mp + b).standard_normal((mp, b))
    p, ldp = e.alloc(mp, b)
    _put(p, a)
    (v, ldv, t, ldt, q2, ldq), ph = e.panel_factor(p, ldp, mp, b)
    ref = orc.qr_tall_pivoted(a)
    assert np.array_equal(ph.cpu().numpy(), ref.perm)
    r = _get(p, mp, b)
    nrm = np.linalg.norm(a)
    assert np.abs(r - ref.r).max() <= 1e-12 * nrm
    # the factors reproduce the panel: A[:, P-hat] = (I - V T V^T) diag(Q2, I) [R; 0]
    vm, tm, qm = _get(v, mp, b), _get(t, b, b), _get(q2, b, b)
    x = np.zeros((mp, b))
    x[:b] = qm @ r[:b]
    x = x - vm @ (tm @ (vm.T @ x))
    assert np.abs(x - a[:, ref.perm]).max() <= 1e-12 * nrm


def test_panel_apply_matches_numpy():
    import torch

    e = _eng()
    mp, b, n2, s, c0 = 900, 64, 300, 37, 5
    rng = np.random.default_rng(2)
    pan = rng.standard_normal((mp, b))
    p, ldp = e.alloc(mp, b)
    _put(p, pan)
    fac, _ = e.panel_factor(p, ldp, mp, b)
    v, ldv, t, ldt, q2, ldq = fac
    vm, tm, qm = _get(v, mp, b), _get(t, b, b), _get(q2, b, b)
    full = rng.standard_normal((s + mp, c0 + n2))
    a, lda = e.alloc(s + mp, c0 + n2)
    _put(a, full)
    e.panel_apply(fac, mp, b, a, lda, s + mp, c0 + n2, s, c0, n2)
    torch.cuda.synchronize()
    x = full[s:, c0:].copy()
    x -= vm @ (tm.T @ (vm.T @ x))
    x[:b] = qm.T @ x[:b]
    got = _get(a, s + mp, c0 + n2)
    assert np.abs(got[s:, c0:] - x).max() <= 1e-12 * np.linalg.norm(full)
    assert np.array_equal(got[:s], full[:s]) and np.array_equal(got[:, :c0], full[:, :c0])


def test_sketch_select_init_pos_ties():
    import randqr_oracle as orc

    e = _eng()
    wdt, n, steps = 40, 500, 32
    y = np.random.default_rng(4).standard_normal((wdt, n))
    y[:, 17] = y[:, 400]  # exact tie: the lower logical position must win
    init = np.random.default_rng(5).permutation(n)
    buf, ld = e.alloc(wdt, n)
    _put(buf, y)
    got = e.select(buf, ld, wdt, n, steps, init)
    order = np.argsort(init, kind="stable")
    yo = np.asfortranarray(y[:, order])
    v = np.zeros((wdt, steps), order="F")
    perm = np.arange(n, dtype=np.int64)
    orc.householder_sweep(yo, v, perm, steps, True)
    assert np.array_equal(got, order[perm[:steps]])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("m,n,b,p", [(800, 800, 64, 8), (700, 530, 96, 10)])
def test_distributed_downdate_world1_nccl(m, n, b, p):
    """The block-cyclic driver's downdated sketch on the GPU step engine (G1 via rq_trinv_upper +
    rq_gemm, Y2 -= G1 R12 per rank) vs the oracle's block_qr_downdate and the single-GPU driver."""
    import torch.distributed as dist

    import randqr_oracle as orc
    from paper_1505_08115_b200 import hqrrp
    from paper_1505_08115_b200.dist import block_qr_distributed

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        a = np.random.default_rng(m + n + 1).standard_normal((m, n))
        cfg = hqrrp.BlockConfig(b, hqrrp.SketchConfig(b, p, 0))
        rng = hqrrp.RngState(3)
        r, perm = block_qr_distributed(a, cfg, rng, sketch="downdate")
        rng1 = hqrrp.RngState(3)
        f = hqrrp.block_qr(a, cfg, rng1, sketch="downdate")
        ref_rng = orc.RngState(3)
        fo = orc.block_qr_downdate(a, orc.BlockConfig(b, orc.SketchConfig(b, p, 0)), ref_rng)
        nrm = np.linalg.norm(a)
        assert np.array_equal(perm, fo.perm())
        assert np.array_equal(perm, f.perm)
        assert np.abs(r - np.triu(fo.r)).max() <= 1e-12 * nrm
        assert np.abs(r - np.triu(f.r)).max() <= 1e-12 * nrm
        assert rng.counter == rng1.counter == ref_rng.counter == m * (b + p)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("m,n,b,p", [(800, 800, 64, 8), (700, 530, 96, 10)])
def test_distributed_world1_nccl_matches_single_gpu(m, n, b, p):
    import torch.distributed as dist

    import randqr_oracle as orc
    from paper_1505_08115_b200 import hqrrp
    from paper_1505_08115_b200.dist import block_qr_distributed

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        a = np.random.default_rng(m + n).standard_normal((m, n))
        cfg = hqrrp.BlockConfig(b, hqrrp.SketchConfig(b, p, 0))
        rng = hqrrp.RngState(3)
        r, perm = block_qr_distributed(a, cfg, rng)
        rng1 = hqrrp.RngState(3)
        f = hqrrp.block_qr(a, cfg, rng1)
        ref_rng = orc.RngState(3)
        fo = orc.block_qr(a, orc.BlockConfig(b, orc.SketchConfig(b, p, 0)), ref_rng)
        nrm = np.linalg.norm(a)
        assert np.array_equal(perm, f.perm)
        assert np.array_equal(perm, fo.perm())
        assert np.abs(r - np.triu(f.r)).max() <= 1e-12 * nrm
        assert np.abs(r - np.triu(fo.r)).max() <= 1e-12 * nrm
        assert rng.counter == rng1.counter == ref_rng.counter
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,steps", [(900, 256), (8800, 256), (9000, 256), (10000, 256), (11000, 128), (13000, 256),
                                     (21500, 96), (24000, 40)])
def test_sketch_select_every_kernel_tier(n, steps):
    """The sketch CPQR picks the reference's pivots in every tier: register-resident
    (n' <= 11840), registers + shared memory (<= ~23k), and the L2-streaming fallback."""
    import randqr_oracle as orc

    e = _eng()
    wdt = 272
    y = np.random.default_rng(n).standard_normal((wdt, n))
    buf, ld = e.alloc(wdt, n)
    _put(buf, y)
    got = e.select(buf, ld, wdt, n, steps, np.arange(n))
    v = np.zeros((wdt, steps), order="F")
    perm = np.arange(n, dtype=np.int64)
    orc.householder_sweep(np.asfortranarray(y), v, perm, steps, True)
    assert np.array_equal(got, perm[:steps])
