import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd())
import paper_1505_08115_b200 as rq  # noqa: E402
from oracle import randqr_oracle as O  # noqa: E402

g = dict(np.load("tests/golden/cfg4_n400.npz"))
a = g["a"]
ours, ref = [], []
rq.block_rrqr(a, rq.BlockConfig(32, rq.SketchConfig(32, 10, 1), "reflectors", True), rq.RngState(1),
              inspect=lambda k, w: ours.append(w))
O.block_rrqr(a, O.BlockConfig(32, O.SketchConfig(32, 10, 1), "reflectors", True), O.RngState(1),
             inspect=lambda k, w: ref.append(w))
for k, (x, y) in enumerate(zip(ours, ref)):
    s = k * 32
    d = np.abs(x - y)
    print(f"panel {k+1}: max|d| {d.max():.2e}  panel block {d[:, s:s+32].max():.2e}  trailing {d[:, s+32:].max() if s+32 < 400 else 0:.2e}"
          f"  diag {np.abs(np.diag(x)[s:s+32] - np.diag(y)[s:s+32]).max():.2e}  dmin {np.diag(y)[s:s+32].min():.1e}")
