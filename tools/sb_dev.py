"""Dev check of the batched sketch CPQR (sketch_batch.cu): pivots vs the oracle on ordinary, tied, rank-deficient
and tiny inputs, then timings.  RQ_SK_BATCH=0 runs the per-step kernel for comparison."""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1505_08115_b200 as rq
from oracle import randqr_oracle as O
from paper_1505_08115_b200.errors import check

eng = rq.Engine()
lib = eng.lib
rng = np.random.default_rng(5)


def dev(x):
    buf, ld = eng.alloc_matrix(*x.shape)
    buf[: x.shape[1], : x.shape[0]].copy_(torch.from_numpy(np.ascontiguousarray(x.T)))
    return buf, ld


def run(y, steps):
    m, n = y.shape
    buf, ld = dev(y)
    ch = torch.full((steps,), -7, dtype=torch.int32, device=eng.device)
    check(lib.rq_test_sketch_cpqr(eng.handle, ctypes.c_void_p(buf.data_ptr()), ld, m, n, steps,
                                  ctypes.c_void_p(ch.data_ptr())))
    torch.cuda.synchronize()
    return ch.cpu().numpy().astype(np.int64)


def case(name, y, steps):
    got = run(y, steps)
    ref = O.qr_column_pivoted(y, steps=steps).perm[:steps]
    ok = np.array_equal(got, ref)
    first = int(np.argmax(got != ref)) if not ok else -1
    print(f"{name}: {'ok' if ok else 'MISMATCH at step %d: got %s ref %s' % (first, got[first:first+4], ref[first:first+4])}",
          flush=True)
    return ok


allok = True
allok &= case("gauss 74x2000/64", rng.standard_normal((74, 2000)), 64)
allok &= case("gauss 272x1000/256", rng.standard_normal((272, 1000)), 256)
allok &= case("gauss 272x300/256", rng.standard_normal((272, 300)), 256)
allok &= case("gauss 40x37/30", rng.standard_normal((40, 37)), 30)
allok &= case("gauss 130x900/100", rng.standard_normal((130, 900)), 100)
y = rng.standard_normal((272, 3000))
y[:, 100] = y[:, 2500]
y[:, 7] = y[:, 2999]
y[:, 1500:1510] = y[:, 20:21]
allok &= case("duplicates 272x3000/256", y, 256)
y = rng.standard_normal((272, 40)) @ rng.standard_normal((40, 2500))
allok &= case("rank 40 272x2500/100", y, 100)
y = np.zeros((80, 500))
allok &= case("zeros 80x500/60", y, 60)
y = rng.standard_normal((80, 500))
y[:, 50:] = 0.0
allok &= case("50 nonzero cols 80x500/70", y, 70)
u, _ = np.linalg.qr(rng.standard_normal((272, 272)))
v, _ = np.linalg.qr(rng.standard_normal((5000, 272)))
y = (u * np.logspace(0, -12, 272)) @ v.T
allok &= case("graded 272x5000/256", y, 256)
allok &= case("gauss 272x10000/256", rng.standard_normal((272, 10000)), 256)
allok &= case("gauss 272x20000/256", rng.standard_normal((272, 20000)), 256)
print("ALL OK" if allok else "FAILURES", flush=True)

for (m, n, steps) in [(272, 20000, 256), (272, 10000, 256), (272, 5000, 256), (272, 1000, 256), (74, 2000, 64)]:
    y0 = rng.standard_normal((m, n))
    buf, ld = dev(y0)
    ch = torch.zeros(steps, dtype=torch.int32, device=eng.device)
    ts = []
    for _ in range(6):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        check(lib.rq_test_sketch_cpqr(eng.handle, ctypes.c_void_p(buf.data_ptr()), ld, m, n, steps,
                                      ctypes.c_void_p(ch.data_ptr())))
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    t = min(ts[1:])
    print(f"sketch cpqr {m}x{n} steps={steps}: {t*1e6:.0f} us ({t*1e6/steps:.2f} us/step)", flush=True)
