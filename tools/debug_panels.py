"""Compare per-panel working matrices (inspect hook) against the oracle (debug aid)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd())
import paper_1505_08115_b200 as rq  # noqa: E402
from oracle import randqr_oracle as O  # noqa: E402

m, n, b, p = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (300, 300, 50, 10)))
a = O.gaussian_matrix(m, n, O.RngState(0))
ours, ref = [], []
f = rq.block_qr(a, rq.BlockConfig(b, rq.SketchConfig(b, p, 0)), rq.RngState(1), inspect=lambda k, w: ours.append(w))
g = O.block_qr(a, O.BlockConfig(b, O.SketchConfig(b, p, 0)), O.RngState(1), inspect=lambda k, w: ref.append(w))
scale = np.linalg.norm(a)
for k, (w1, w2) in enumerate(zip(ours, ref)):
    d = np.abs(w1 - w2)
    s = min((k + 1) * b, n)
    print(f"panel {k+1}: max|d|/|A| = {d.max()/scale:.2e}  panel-cols {d[:, k*b:s].max()/scale:.2e} "
          f"trail {d[:, s:].max()/scale if s < n else 0:.2e}")
print("perm equal:", np.array_equal(f.perm, g.perm()))
print("ours", f.perm[:12])
print("ref ", g.perm()[:12])
