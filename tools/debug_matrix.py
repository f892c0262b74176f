"""Which (n, b, p) configs diverge from the oracle, and at which panel (debug aid)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd())
import paper_1505_08115_b200 as rq  # noqa: E402
from oracle import randqr_oracle as O  # noqa: E402

eng = rq.Engine()
for n in (64, 100, 128, 200, 300):
    for b in (8, 16, 24, 32, 40, 50, 64):
        for p in (0, 4):
            if b >= n:
                continue
            a = O.gaussian_matrix(n, n, O.RngState(0))
            ours, ref = [], []
            try:
                rq.block_qr(a, rq.BlockConfig(b, rq.SketchConfig(b, p, 0)), rq.RngState(1),
                            inspect=lambda k, w: ours.append(w), engine=eng)
                O.block_qr(a, O.BlockConfig(b, O.SketchConfig(b, p, 0)), O.RngState(1),
                           inspect=lambda k, w: ref.append(w))
            except ValueError:
                continue
            scale = np.linalg.norm(a)
            bad = [k + 1 for k, (x, y) in enumerate(zip(ours, ref)) if np.abs(x - y).max() > 1e-12 * scale]
            print(f"n={n} b={b} p={p}: {'OK' if not bad else 'first bad panel %d of %d' % (bad[0], len(ref))}")
