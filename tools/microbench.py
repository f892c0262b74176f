"""Time the serial kernels in isolation through the C-ABI test hooks (debug/perf aid)."""
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
st = eng.stream


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def dev(x):
    buf, ld = eng.alloc_matrix(*x.shape)
    buf[: x.shape[1], : x.shape[0]].copy_(torch.from_numpy(np.ascontiguousarray(x.T)))
    return buf, ld


rng = np.random.default_rng(0)
which = sys.argv[1:] or ["sweep", "sketch", "leaf"]
if "sweep" in which:
    for (m, n, steps) in [(256, 256, 256), (128, 128, 128), (64, 64, 64)]:
        a0 = rng.standard_normal((m, n))
        buf, ld = dev(a0)
        work, _ = eng.alloc_matrix(m, n)
        v, ldv = eng.alloc_matrix(m, steps)
        perm = torch.arange(n, dtype=torch.int64, device=eng.device)

        def run():
            work.copy_(buf)
            v.zero_()
            check(lib.rq_householder_sweep(eng.handle, ctypes.c_void_p(work.data_ptr()), m, n, ld,
                                           ctypes.c_void_p(v.data_ptr()), ldv, ctypes.c_void_p(perm.data_ptr()),
                                           steps, 1))
        ms = timeit(run)
        print(f"cpqr sweep {m}x{n} steps={steps}: {ms*1e3:.0f} us  ({ms*1e3/steps:.2f} us/step)")
if "sketch" in which:
    for _ in [0]:
        for (m, n, steps) in [(272, 40000, 256), (272, 20000, 256), (272, 11800, 256), (272, 10000, 256), (272, 5000, 256), (272, 1000, 256), (74, 2000, 64)]:
            y0 = rng.standard_normal((m, n))
            buf, ld = dev(y0)
            work, _ = eng.alloc_matrix(m, n)
            ch = torch.zeros(steps, dtype=torch.int32, device=eng.device)

            def run():
                work.copy_(buf)
                check(lib.rq_test_sketch_cpqr(eng.handle, ctypes.c_void_p(work.data_ptr()), ld, m, n, steps,
                                              ctypes.c_void_p(ch.data_ptr())))
            ms = timeit(run)
            print(f"sketch cpqr {m}x{n} steps={steps}: {ms*1e3:.0f} us  ({ms*1e3/steps:.2f} us/step)")
if "leaf" in which:
    for (mm, w) in [(10000, 16), (10000, 32), (5000, 32), (2000, 32), (40000, 8)]:
        a0 = rng.standard_normal((mm, w))
        buf, ld = dev(a0)
        work, _ = eng.alloc_matrix(mm, w)
        v, ldv = eng.alloc_matrix(mm, w)
        t, ldt = eng.alloc_matrix(32, 32)

        def run():
            work.copy_(buf)
            check(lib.rq_test_leaf_qr(eng.handle, ctypes.c_void_p(work.data_ptr()), ld, mm, w,
                                      ctypes.c_void_p(v.data_ptr()), ldv, ctypes.c_void_p(t.data_ptr()), ldt))
        try:
            ms = timeit(run)
            print(f"leaf {mm}x{w}: {ms*1e3:.0f} us  ({ms*1e3/w:.2f} us/column)")
        except Exception as e:  # width not supported at this height
            print(f"leaf {mm}x{w}: {e}")
if "stamps" in which:
    m = n = 256
    a0 = rng.standard_normal((m, n))
    buf, ld = dev(a0)
    v, ldv = eng.alloc_matrix(m, n)
    perm = torch.arange(n, dtype=torch.int64, device=eng.device)
    check(lib.rq_test_debug_timing(1, None, 0))
    check(lib.rq_householder_sweep(eng.handle, ctypes.c_void_p(buf.data_ptr()), m, n, ld,
                                   ctypes.c_void_p(v.data_ptr()), ldv, ctypes.c_void_p(perm.data_ptr()), n, 1))
    torch.cuda.synchronize()
    h = np.zeros(512, dtype=np.uint64)
    check(lib.rq_test_debug_timing(0, h.ctypes.data_as(ctypes.c_void_p), 512))
    h = h.reshape(64, 8).astype(np.int64)
    d = np.diff(h[5:60], axis=1)
    print("cluster sweep phase cycles (median over steps 5..60):")
    names = ["A:update+score", "sync1", "argmax+pushkey+sync2", "stage", "cluster barrier", "F+G: winner, pull, u",
             "H + sync3"]
    for k, nm in enumerate(names):
        print(f"  {nm:18s} {int(np.median(d[:, k])):6d}")
    print("  step total        ", int(np.median(h[6:60, 0] - h[5:59, 0])))

if "skstamps" in which:
    m, n, steps = 272, int(os.environ.get("SKN", "10000")), 256
    y0 = rng.standard_normal((m, n))
    buf, ld = dev(y0)
    ch = torch.zeros(steps, dtype=torch.int32, device=eng.device)
    check(lib.rq_test_debug_timing(1, None, 0))
    check(lib.rq_test_sketch_cpqr(eng.handle, ctypes.c_void_p(buf.data_ptr()), ld, m, n, steps,
                                  ctypes.c_void_p(ch.data_ptr())))
    torch.cuda.synchronize()
    h = np.zeros(512, dtype=np.uint64)
    check(lib.rq_test_debug_timing(0, h.ctypes.data_as(ctypes.c_void_p), 512))
    h = h.reshape(64, 8).astype(np.int64)
    d = np.diff(h[5:60, :7], axis=1)
    print(f"sketch cpqr phase cycles n={n} (median over steps 5..60):")
    names = ["A: apply+score", "sync", "B: cta best + column", "C: arrive/last-reduces/poll", "E: u+pos", "-"]
    for k, nm in enumerate(names):
        print(f"  {nm:20s} {int(np.median(d[:, k])):6d}")
    print("  step total          ", int(np.median(h[6:60, 0] - h[5:59, 0])))

if "gemm" in which or "gemm_tn" in which:
    def gemm_case(mm, M, N, K, label):
        A = torch.randn((K, M) if not mm else (M, K), dtype=torch.float64, device=eng.device)
        B = torch.randn((K, N), dtype=torch.float64, device=eng.device)
        C = torch.randn((M, N), dtype=torch.float64, device=eng.device)
        # column-major views: storage (cols, rows)
        As = A.T.contiguous() if False else A  # storage as (cols, ld)
        a_rows, a_cols = (M, K) if mm else (K, M)
        abuf, lda = eng.alloc_matrix(a_rows, a_cols)
        bbuf, ldb = eng.alloc_matrix(K, N)
        cbuf, ldc = eng.alloc_matrix(M, N)
        abuf.normal_(); bbuf.normal_(); cbuf.normal_()

        def run():
            check(lib.rq_test_gemm(eng.handle, int(mm), M, N, K, ctypes.c_void_p(abuf.data_ptr()), lda, a_rows, a_cols,
                                   0, 0, ctypes.c_void_p(bbuf.data_ptr()), ldb, K, N, 0, 0,
                                   ctypes.c_void_p(cbuf.data_ptr()), ldc, -1.0, 1.0))
        ms = timeit(run, reps=5)
        print(f"gemm {label:28s} M={M} N={N} K={K}: {ms*1e3:8.0f} us  {2*M*N*K/ms/1e9:6.2f} TF/s")
if "gemm" in which:
    gemm_case(1, 10000, 10000, 256, "NN  A2 -= V W2")
    gemm_case(0, 256, 10000, 10000, "TN  W = V^T A2")
    gemm_case(0, 272, 10000, 10000, "TN  Yt = Om^T X (sketch)")
    gemm_case(0, 256, 256, 10000, "TN  Gram V^T V")
    gemm_case(1, 5000, 5000, 256, "NN  half size")
    gemm_case(0, 4096, 4096, 4096, "TN  square 4096")
if "gemm_tn" in which:
    for nn in (9600, 12000, 16000, 20000, 30000):
        gemm_case(0, 256, nn, nn, "TN  W = V^T A2")
if "gemm_nn" in which:
    M, N, K = 10000, 10000, 256
    abuf, lda = eng.alloc_matrix(M, K)
    bbuf, ldb = eng.alloc_matrix(K, N)
    cbuf, ldc = eng.alloc_matrix(M, N)
    abuf.normal_(); bbuf.normal_(); cbuf.normal_()
    for _ in range(2):
        check(lib.rq_test_gemm(eng.handle, 1, M, N, K, ctypes.c_void_p(abuf.data_ptr()), lda, M, K, 0, 0,
                               ctypes.c_void_p(bbuf.data_ptr()), ldb, K, N, 0, 0, ctypes.c_void_p(cbuf.data_ptr()),
                               ldc, -1.0, 1.0))
    torch.cuda.synchronize()

if "gemm_tn" in which:
    # W = V^T A2 at n = 10k, as the trailing update issues it (split-K workspace from the engine)
    M, N, K = 256, 10000, 10000
    abuf, lda = eng.alloc_matrix(K, M)
    bbuf, ldb = eng.alloc_matrix(K, N)
    cbuf, ldc = eng.alloc_matrix(M, N)
    abuf.normal_(); bbuf.normal_(); cbuf.normal_()
    for _ in range(2):
        check(lib.rq_test_gemm(eng.handle, 0, M, N, K, ctypes.c_void_p(abuf.data_ptr()), lda, K, M, 0, 0,
                               ctypes.c_void_p(bbuf.data_ptr()), ldb, K, N, 0, 0, ctypes.c_void_p(cbuf.data_ptr()),
                               ldc, 1.0, 0.0))
    torch.cuda.synchronize()

if "leafstamps" in which:
    mm, w = int(os.environ.get("LEAFM", "10000")), 16
    a0 = rng.standard_normal((mm, w))
    buf, ld = dev(a0)
    v, ldv = eng.alloc_matrix(mm, w)
    t, ldt = eng.alloc_matrix(32, 32)
    check(lib.rq_test_debug_timing(2, None, 0))
    check(lib.rq_test_leaf_qr(eng.handle, ctypes.c_void_p(buf.data_ptr()), ld, mm, w,
                              ctypes.c_void_p(v.data_ptr()), ldv, ctypes.c_void_p(t.data_ptr()), ldt))
    torch.cuda.synchronize()
    h = np.zeros(512, dtype=np.uint64)
    check(lib.rq_test_debug_timing(0, h.ctypes.data_as(ctypes.c_void_p), -512))
    h = h.reshape(64, 8).astype(np.int64)
    d = np.diff(h[2:14], axis=1)
    names = ["apply+partials", "reduce-scatter", "sync", "cta sum+push", "cluster barrier", "T+reflector(w0)", "sync"]
    print(f"leaf phase cycles mm={mm} w={w} (median over columns 2..13):")
    for k, nm in enumerate(names):
        print(f"  {nm:18s} {int(np.median(d[:, k])):6d}")
    print("  column total      ", int(np.median(h[3:14, 0] - h[2:13, 0])))
if "leaf1" in which:
    mm, w = int(os.environ.get("LEAFM", "10000")), 16
    a0 = rng.standard_normal((mm, w))
    buf, ld = dev(a0)
    v, ldv = eng.alloc_matrix(mm, w)
    t, ldt = eng.alloc_matrix(32, 32)
    for _ in range(2):
        check(lib.rq_test_leaf_qr(eng.handle, ctypes.c_void_p(buf.data_ptr()), ld, mm, w,
                                  ctypes.c_void_p(v.data_ptr()), ldv, ctypes.c_void_p(t.data_ptr()), ldt))
    torch.cuda.synchronize()

if "prof" in which:
    # one leaf (10000 x 16) and one sketch CPQR (272 x 10000, 256 steps), each run twice: the
    # second launches are the ones an `ncu -k regex:"leaf_reg|sketch_reg" -s 1` capture reads
    mm, w = 10000, 16
    a0 = rng.standard_normal((mm, w))
    lbuf, lld = dev(a0)
    v, ldv = eng.alloc_matrix(mm, w)
    t, ldt = eng.alloc_matrix(32, 32)
    m, n, steps = 272, 10000, 256
    y0 = rng.standard_normal((m, n))
    ybuf, yld = dev(y0)
    ywork, _ = eng.alloc_matrix(m, n)
    ch = torch.zeros(steps, dtype=torch.int32, device=eng.device)
    for _ in range(2):
        lw = lbuf.clone()
        check(lib.rq_test_leaf_qr(eng.handle, ctypes.c_void_p(lw.data_ptr()), lld, mm, w,
                                  ctypes.c_void_p(v.data_ptr()), ldv, ctypes.c_void_p(t.data_ptr()), ldt))
        ywork.copy_(ybuf)
        check(lib.rq_test_sketch_cpqr(eng.handle, ctypes.c_void_p(ywork.data_ptr()), yld, m, n, steps,
                                      ctypes.c_void_p(ch.data_ptr())))
    torch.cuda.synchronize()
    print("prof ok")

if "wy" in which:
    # WY update of one leaf (w = 16) on the rest of the panel: whole-GPU kernel vs 16-CTA cluster
    for (mm, nr) in [(20000, 240), (20000, 120), (10000, 240), (10000, 120), (40000, 120)]:
        w = 16
        a0 = torch.randn((nr, mm + (mm & 1)), dtype=torch.float64, device=eng.device)
        vv = torch.randn((w, mm + (mm & 1)), dtype=torch.float64, device=eng.device) / mm ** 0.5
        tt = torch.triu(torch.randn((32, 32), dtype=torch.float64, device=eng.device)).T.contiguous()
        work = a0.clone()
        res = {}
        for cl in (0, 1):
            def run():
                check(lib.rq_test_wy_update(eng.handle, cl, ctypes.c_void_p(work.data_ptr()), mm + (mm & 1), mm, nr,
                                            ctypes.c_void_p(vv.data_ptr()), mm + (mm & 1),
                                            ctypes.c_void_p(tt.data_ptr()), 32, w))
            try:
                work.copy_(a0)
                run()
                torch.cuda.synchronize()
                res[cl] = work.clone()
                ms = timeit(run, reps=5)
                gb = 3.0 * mm * nr * 8 / 1e9
                print(f"wy {'cluster' if cl else 'grid   '} mm={mm} nr={nr}: {ms*1e3:7.1f} us  {gb/(ms*1e-3):6.0f} GB/s")
            except Exception as e:
                print(f"wy cl={cl} mm={mm} nr={nr}: {e}")
        if 0 in res and 1 in res:
            ref = a0.clone()
            print("   max |grid - cluster| / max|A|:", float((res[0] - res[1]).abs().max() / a0.abs().max()))
