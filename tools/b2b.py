"""Back-to-back vs synchronised factorizations (n = 10k, downdated sketch): device ms per factorization."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch

import paper_1505_08115_b200 as rq
from paper_1505_08115_b200 import _lib
from paper_1505_08115_b200.errors import check

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
b, p = 256, 16
smode = sys.argv[2] if len(sys.argv) > 2 else "default"
if smode == "default":
    eng = rq.Engine()
elif smode == "new":
    eng = rq.Engine(0, stream=torch.cuda.Stream())
else:  # "hi": a created stream of the highest priority
    eng = rq.Engine(0, stream=torch.cuda.Stream(priority=-1))
stream = eng.stream
print("stream mode", smode)
with torch.cuda.stream(stream):
    a0, ld = rq.gaussian_matrix_device(n, n, rq.RngState(0), engine=eng)
    work = torch.empty_like(a0)
    perm = torch.empty(n, dtype=torch.int64, device=a0.device)
cfg = _lib.rq_config(b, p, 0, -1, _lib.RQ_PIVOT_PERMUTATION, 0, _lib.RQ_SKETCH_DOWNDATE, 0)


def step(copy=True):
    if copy:
        with torch.cuda.stream(stream):
            work.copy_(a0)
    ctr = ctypes.c_uint64(0)
    check(eng.lib.rq_factorize(eng.handle, ctypes.byref(cfg), n, n, ctypes.c_void_p(work.data_ptr()), ld,
                               ctypes.c_uint64(1), ctypes.byref(ctr), ctypes.c_void_p(perm.data_ptr())))


for _ in range(3):
    step()
torch.cuda.synchronize()
for mode in ("sync", "b2b"):
    K = 5
    tot = 0.0
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    if mode == "b2b":
        e0.record(stream)
        h0 = time.perf_counter()
        for _ in range(K):
            step()
        h = (time.perf_counter() - h0) / K * 1e3
        e1.record(stream)
        torch.cuda.synchronize()
        print(f"{mode}: {e0.elapsed_time(e1) / K:.2f} ms per factorization (host enqueue {h:.1f} ms)")
    else:
        hs = 0.0
        for _ in range(K):
            with torch.cuda.stream(stream):
                work.copy_(a0)
            torch.cuda.synchronize()
            e0.record(stream)
            h0 = time.perf_counter()
            step(copy=False)
            hs += time.perf_counter() - h0
            e1.record(stream)
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
        print(f"{mode}: {tot / K:.2f} ms per factorization (host enqueue {hs / K * 1e3:.1f} ms)")
