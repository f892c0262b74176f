"""Isolate the sketch CPQR: oracle Y^T through our sweep vs oracle pivots (debug aid)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd())
import paper_1505_08115_b200 as rq  # noqa: E402
from oracle import randqr_oracle as O  # noqa: E402

eng = rq.Engine()
for (n, b, p) in [(100, 40, 4), (100, 32, 4), (100, 40, 0), (128, 50, 4), (300, 64, 4), (64, 20, 4), (64, 20, 24)]:
    a = O.gaussian_matrix(n, n, O.RngState(0))
    y = O.build_sketch(a, O.SketchConfig(b, p, 0), O.RngState(1))
    yt = np.asfortranarray(y.T)
    ref = O.qr_column_pivoted(yt, steps=b)
    a1 = yt.copy(order="F")
    v = np.zeros((b + p, b), order="F")
    perm = np.arange(n, dtype=np.int64)
    rq.householder_sweep(a1, v, perm, b, True, engine=eng)
    nd = np.nonzero(perm[:b] != ref.perm[:b])[0]
    print(n, b, p, "pivots equal" if len(nd) == 0 else f"first diff at step {nd[0]}: ours {perm[nd[0]]} ref {ref.perm[nd[0]]}",
          "max|dR|", np.abs(a1[:, :b] - ref.r[:, :b]).max())
