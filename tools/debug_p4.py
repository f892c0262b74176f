import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd())
import paper_1505_08115_b200 as rq  # noqa: E402
from oracle import randqr_oracle as O  # noqa: E402

n, b, p = 100, 40, 4
a = O.gaussian_matrix(n, n, O.RngState(0))
ours, ref = [], []
f = rq.block_qr(a, rq.BlockConfig(b, rq.SketchConfig(b, p, 0)), rq.RngState(1), inspect=lambda k, w: ours.append(w))
g = O.block_qr(a, O.BlockConfig(b, O.SketchConfig(b, p, 0)), O.RngState(1), inspect=lambda k, w: ref.append(w))
print("perm[:b] same set:", set(f.perm[:b]) == set(g.perm()[:b]))
print("ours", f.perm[:b])
print("ref ", g.perm()[:b])
w1, w2 = ours[0], ref[0]
d = np.abs(w1 - w2)
print("panel cols diff", d[:, :b].max(), "trail", d[:, b:].max())
print("diag ours", np.diag(w1)[:8])
print("diag ref ", np.diag(w2)[:8])
# columns of trailing: compare as sets by matching
