"""Rate of the fp64 DMMA GEMM on the trailing-update shapes, with and without the C read (beta),
and at longer K (mainloop share).  Tuning aid: python tools/gemm_probe.py"""
import ctypes
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_1505_08115_b200 as rq  # noqa: E402
from paper_1505_08115_b200.errors import check  # noqa: E402

eng = rq.Engine()
lib, st = eng.lib, eng.stream


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def case(mm, M, N, K, beta, label):
    a_rows, a_cols = (M, K) if mm else (K, M)
    abuf, lda = eng.alloc_matrix(a_rows, a_cols)
    bbuf, ldb = eng.alloc_matrix(K, N)
    cbuf, ldc = eng.alloc_matrix(M, N)
    abuf.normal_()
    bbuf.normal_()
    cbuf.normal_()

    def run():
        check(lib.rq_test_gemm(eng.handle, int(mm), M, N, K, ctypes.c_void_p(abuf.data_ptr()), lda, a_rows, a_cols,
                               0, 0, ctypes.c_void_p(bbuf.data_ptr()), ldb, K, N, 0, 0,
                               ctypes.c_void_p(cbuf.data_ptr()), ldc, -1.0, beta))
    ms = timeit(run)
    print(f"{label:24s} M={M} N={N} K={K} beta={beta}: {ms*1e3:8.1f} us  {2*M*N*K/ms/1e9:6.2f} TF/s", flush=True)
    del abuf, bbuf, cbuf


for K in (256, 512, 1024):
    for beta in (1.0, 0.0):
        case(1, 10000, 10000, K, beta, "NN A2 -= V W2")
case(1, 20000, 20000, 256, 1.0, "NN 20k")
case(0, 256, 10000, 10000, 0.0, "TN W = V^T A2")
