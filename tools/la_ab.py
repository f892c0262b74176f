"""A/B of the look-ahead (RQ_LOOKAHEAD, read at first use) in the downdated-sketch driver:
device time of block_qr on an n x n Gaussian (no profiling events), plus the permutation and
|diag(R)| saved to gpurun_out/la_<tag>_<n>.npz so runs with and without it can be compared.
Usage: RQ_LOOKAHEAD=k python tools/la_ab.py n tag"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1505_08115_b200 as rq  # noqa: E402
from paper_1505_08115_b200 import _lib  # noqa: E402
from paper_1505_08115_b200.errors import check  # noqa: E402

n = int(sys.argv[1])
tag = sys.argv[2] if len(sys.argv) > 2 else "x"
b, p = 256, 16
stream = torch.cuda.Stream()
eng = rq.Engine(0, stream=stream)
with torch.cuda.stream(stream):
    a0, ld = rq.gaussian_matrix_device(n, n, rq.RngState(0), engine=eng)
    work, _ = eng.alloc_matrix(n, n)
    perm = torch.empty(n, dtype=torch.int64, device=eng.device)
cfg = _lib.rq_config(b, p, 0, -1, _lib.RQ_PIVOT_PERMUTATION, 0, _lib.RQ_SKETCH_DOWNDATE, 0)


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
k = 3
e0.record(stream)
for _ in range(k):
    step()
e1.record(stream)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / k
d = torch.diagonal(work[:n, :n]).abs().cpu().numpy()
os.makedirs("gpurun_out", exist_ok=True)
np.savez(f"gpurun_out/la_{tag}_{n}.npz", perm=perm.cpu().numpy(), d=d)
print(f"n={n} RQ_LOOKAHEAD={os.environ.get('RQ_LOOKAHEAD', '1')} {ms:.1f} ms "
      f"{4 / 3 * n ** 3 / ms / 1e9:.2f} TFLOP/s launches={eng.launches}", flush=True)
