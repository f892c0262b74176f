"""A/B of the in-panel overlap modes (RQ_OVERLAP, read at first use): device time of
block_qr on n x n Gaussian, no profiling events.  Usage: RQ_OVERLAP=k python tools/overlap_ab.py n"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_1505_08115_b200 as rq  # noqa: E402
from paper_1505_08115_b200 import _lib  # noqa: E402
from paper_1505_08115_b200.errors import check  # noqa: E402

n = int(sys.argv[1])
b, p = 256, 16
stream = torch.cuda.Stream()
eng = rq.Engine(0, stream=stream)
with torch.cuda.stream(stream):
    a0, ld = rq.gaussian_matrix_device(n, n, rq.RngState(0), engine=eng)
    work, _ = eng.alloc_matrix(n, n)
    perm = torch.empty(n, dtype=torch.int64, device=eng.device)
cfg = _lib.rq_config(b, p, 0, -1, _lib.RQ_PIVOT_PERMUTATION, 0, _lib.RQ_SKETCH_FRESH, 0)


def step():
    with torch.cuda.stream(stream):
        work.copy_(a0)
    ctr = ctypes.c_uint64(0)
    check(eng.lib.rq_factorize(eng.handle, ctypes.byref(cfg), n, n, ctypes.c_void_p(work.data_ptr()), ld,
                               ctypes.c_uint64(1), ctypes.byref(ctr), ctypes.c_void_p(perm.data_ptr())))


for _ in range(2):
    step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for _ in range(3):
    step()
e1.record(stream)
torch.cuda.synchronize()
print(f"RQ_OVERLAP={os.environ.get('RQ_OVERLAP', '1')} n={n} ms={e0.elapsed_time(e1) / 3:.1f} perm0={perm[:4].tolist()}")
