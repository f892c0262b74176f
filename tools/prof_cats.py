"""Per-class kernel time of one profiled factorization (CUDA events around every launch; the
classes overlap in time).  Usage: python tools/prof_cats.py n [downdate|fresh]"""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import paper_1505_08115_b200 as rq  # noqa: E402
from paper_1505_08115_b200 import _lib  # noqa: E402
from paper_1505_08115_b200.errors import check  # noqa: E402

n = int(sys.argv[1])
mode = _lib.RQ_SKETCH_FRESH if len(sys.argv) > 2 and sys.argv[2] == "fresh" else _lib.RQ_SKETCH_DOWNDATE
stream = torch.cuda.Stream()
eng = rq.Engine(0, stream=stream)
with torch.cuda.stream(stream):
    a0, ld = rq.gaussian_matrix_device(n, n, rq.RngState(0), engine=eng)
    work, _ = eng.alloc_matrix(n, n)
    perm = torch.empty(n, dtype=torch.int64, device=eng.device)
cfg = _lib.rq_config(256, 16, 0, -1, _lib.RQ_PIVOT_PERMUTATION, 0, mode, 0)


def step():
    with torch.cuda.stream(stream):
        work.copy_(a0)
    ctr = ctypes.c_uint64(0)
    check(eng.lib.rq_factorize(eng.handle, ctypes.byref(cfg), n, n, ctypes.c_void_p(work.data_ptr()), ld,
                               ctypes.c_uint64(1), ctypes.byref(ctr), ctypes.c_void_p(perm.data_ptr())))


step()
torch.cuda.synchronize()
check(eng.lib.rq_set_profiling(eng.handle, 1))
step()
torch.cuda.synchronize()
for c, name in enumerate(["trailing_gemm", "other_gemm", "sketch_cpqr", "panel_leaf", "other", "small_cpqr",
                          "sketch_gemm", "panel_gemm", "tfactor"]):
    t, f, k = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
    check(eng.lib.rq_profile_read(eng.handle, c, ctypes.byref(t), ctypes.byref(f), ctypes.byref(k)))
    print(f"{name:14s} {t.value:9.2f} ms  launches {k.value:6d}  {f.value / max(t.value, 1e-9) / 1e9:7.2f} TFLOP/s")
