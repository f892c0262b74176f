"""Sketch CPQR in isolation under different process states (default stream, a PyTorch stream, PyTorch's stream
pool merely existing, k raw streams created first): the per-step time used to flip between ~4.55 and ~5.4 us
with the address cudaMalloc gave the winner record; with the placement calibration (driver.cu
place_sketch_words, RQ_SK_PLACE_CAL=2 prints it) every state runs at the fast speed."""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1505_08115_b200 as rq
from paper_1505_08115_b200.errors import check

mode = sys.argv[1] if len(sys.argv) > 1 else "default"
if mode == "default":
    eng = rq.Engine()
elif mode == "default_pool":  # default stream, but torch's stream pool exists (one unused torch stream)
    _unused = torch.cuda.Stream()
    eng = rq.Engine()
elif mode == "default_pool_hi":
    _unused = torch.cuda.Stream(priority=-1)
    eng = rq.Engine()
elif mode.startswith("dummies"):  # default stream + k raw streams of mixed priorities
    from cuda import cudart
    torch.zeros(1, device="cuda")
    keep = [cudart.cudaStreamCreateWithPriority(cudart.cudaStreamNonBlocking, -(i % 2))[1] for i in range(int(mode[7:]))]
    eng = rq.Engine()
elif mode == "new":
    eng = rq.Engine(0, stream=torch.cuda.Stream())
elif mode == "hi":
    eng = rq.Engine(0, stream=torch.cuda.Stream(priority=-1))
else:
    from cuda import cudart
    torch.cuda.init()
    torch.zeros(1, device="cuda")
    if mode == "blocking":
        err, st = cudart.cudaStreamCreate()
    elif mode == "nonblocking":
        err, st = cudart.cudaStreamCreateWithFlags(cudart.cudaStreamNonBlocking)
    elif mode == "blocking_hi":
        err, st = cudart.cudaStreamCreateWithPriority(cudart.cudaStreamDefault, -5)
    elif mode == "perthread":
        err, st = 0, 2  # cudaStreamPerThread
    eng = rq.Engine(0, stream=torch.cuda.ExternalStream(int(st)))
torch.cuda.set_stream(eng.stream)
rng = np.random.default_rng(5)
for (m, n, steps) in [(272, 10000, 256), (272, 1000, 256)]:
    y0 = rng.standard_normal((m, n))
    buf, ld = eng.alloc_matrix(m, n)
    buf[:n, :m].copy_(torch.from_numpy(np.ascontiguousarray(y0.T)))
    ch = torch.zeros(steps, dtype=torch.int32, device=eng.device)
    ts = []
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    for _ in range(6):
        torch.cuda.synchronize()
        e0.record(eng.stream)
        check(eng.lib.rq_test_sketch_cpqr(eng.handle, ctypes.c_void_p(buf.data_ptr()), ld, m, n, steps,
                                          ctypes.c_void_p(ch.data_ptr())))
        e1.record(eng.stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = min(ts[1:])
    print(f"{mode}: sketch cpqr {m}x{n} steps={steps}: {t*1e3:.0f} us ({t*1e3/steps:.2f} us/step)", flush=True)
