"""Small-shape runs of every serial kernel and one small factorization per mode, for
compute-sanitizer (racecheck / synccheck / memcheck; one tool per gpurun call):

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py

Kernels: sketch_reg_kernel (register tier, LL grid exchange), sweep_reg_kernel (cluster CPQR,
st.async pushes), leaf_reg_kernel (cluster leaf QR), wy_cluster_kernel and wy_update_kernel,
the Jacobi panel SVD, then block_qr (fresh + downdate look-ahead) and block_rrqr end to end.
"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_1505_08115_b200 as rq  # noqa: E402
from paper_1505_08115_b200.errors import check  # noqa: E402

eng = rq.Engine()
lib = eng.lib
rng = np.random.default_rng(0)


def dev(x):
    buf, ld = eng.alloc_matrix(*x.shape)
    buf[: x.shape[1], : x.shape[0]].copy_(torch.from_numpy(np.ascontiguousarray(x.T)))
    return buf, ld


def p(t):
    return ctypes.c_void_p(t.data_ptr())


# sketch CPQR, register tier (two grid sizes)
for (m, n, steps) in [(272, 1000, 64), (74, 600, 32)]:
    y, ld = dev(rng.standard_normal((m, n)))
    ch = torch.zeros(steps, dtype=torch.int32, device=eng.device)
    check(lib.rq_test_sketch_cpqr(eng.handle, p(y), ld, m, n, steps, p(ch)))
# cluster CPQR sweep (b x b)
for k in (64, 128):
    a, ld = dev(rng.standard_normal((k, k)))
    v, ldv = eng.alloc_matrix(k, k)
    v.zero_()
    perm = torch.arange(k, dtype=torch.int64, device=eng.device)
    check(lib.rq_householder_sweep(eng.handle, p(a), k, k, ld, p(v), ldv, p(perm), k, 1))
# leaf QR (cluster)
for (mm, w) in [(2000, 16), (600, 32)]:
    a, ld = dev(rng.standard_normal((mm, w)))
    v, ldv = eng.alloc_matrix(mm, w)
    t, ldt = eng.alloc_matrix(32, 32)
    check(lib.rq_test_leaf_qr(eng.handle, p(a), ld, mm, w, p(v), ldv, p(t), ldt))
# WY updates: cluster and whole-GPU kernels
for cl in (1, 0):
    mm, nr, w = 1500, 100, 16
    a, ld = dev(rng.standard_normal((mm, nr)))
    vv = np.tril(rng.standard_normal((mm, w)))
    vbuf, ldv = dev(vv)
    tt, ldt = dev(np.triu(rng.standard_normal((w, w))))
    check(lib.rq_test_wy_update(eng.handle, cl, p(a), ld, mm, nr, p(vbuf), ldv, p(tt), ldt, w))
torch.cuda.synchronize()
# end to end, every mode (the look-ahead schedule with the off-chain CPQR included)
a = rng.standard_normal((900, 800))
cfg = rq.BlockConfig(128, rq.SketchConfig(128, 10, 0))
rq.block_qr(a, cfg, rq.RngState(1)).expand_q()
rq.block_qr(a, cfg, rq.RngState(1), sketch="downdate").expand_q()
rq.block_qr(a[:300, :300], rq.BlockConfig(48, rq.SketchConfig(48, 8, 1), "reflectors"), rq.RngState(2)).expand_p()
rq.block_rrqr(a[:300, :300], rq.BlockConfig(48, rq.SketchConfig(48, 10, 1), "reflectors", True),
              rq.RngState(3)).expand_p()
torch.cuda.synchronize()
print("sanitize cases done")
