"""Bisect helper: one small factorization per call, with a deadline (run under timeout)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_1505_08115_b200 as rq
n, b, p = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
a = np.random.default_rng(0).standard_normal((n, n))
t0 = time.time()
f = rq.block_qr(a, rq.BlockConfig(b, rq.SketchConfig(b, p, 0)), rq.RngState(1))
print("done", n, b, p, f.perm[:5], round(time.time() - t0, 2), flush=True)
