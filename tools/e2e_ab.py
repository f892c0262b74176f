"""Time the host-buffer entry rq_factorize_host (H2D of A, factorization, R streamed back) for
the sketch modes / look-ahead flag.  Usage: python tools/e2e_ab.py n"""
import ctypes
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1505_08115_b200 as rq  # noqa: E402
from paper_1505_08115_b200 import _lib  # noqa: E402
from paper_1505_08115_b200.errors import check  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
b, p = 256, 16
import os
stream = torch.cuda.Stream() if os.environ.get('E2E_STREAM', '1') == '1' else None
eng = rq.Engine(0, stream=stream) if stream is not None else rq.Engine(0)
a0, ld = rq.gaussian_matrix_device(n, n, rq.RngState(0), engine=eng)
ha = torch.empty((n, ld), dtype=torch.float64, pin_memory=True)
ha.copy_(a0.cpu())
hr = torch.empty((n, ld), dtype=torch.float64, pin_memory=True)
hp = torch.empty(n, dtype=torch.int64, pin_memory=True)
for name, mode, flags in [("downdate+LA", _lib.RQ_SKETCH_DOWNDATE, 0),
                          ("downdate", _lib.RQ_SKETCH_DOWNDATE, _lib.RQ_FLAG_NO_LOOKAHEAD),
                          ("fresh", _lib.RQ_SKETCH_FRESH, 0)]:
    cfg = _lib.rq_config(b, p, 0, -1, _lib.RQ_PIVOT_PERMUTATION, 0, mode, flags)

    def step(host=True):
        ctr = ctypes.c_uint64(0)
        check(eng.lib.rq_factorize_host(eng.handle, ctypes.byref(cfg), n, n, ctypes.c_void_p(ha.data_ptr()), ld,
                                        ctypes.c_uint64(1), ctypes.byref(ctr),
                                        ctypes.c_void_p(hr.data_ptr() if host else None), ld,
                                        ctypes.c_void_p(hp.data_ptr())))

    for host in (True, False):
        step(host)
        t0 = time.perf_counter()
        for _ in range(3):
            step(host)
        dt = (time.perf_counter() - t0) / 3
        print(f"{name:12s} R to host={host}: {dt*1e3:.1f} ms  {4/3*n**3/dt/1e12:.2f} TFLOP/s", flush=True)
