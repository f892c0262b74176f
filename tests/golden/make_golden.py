"""Generate golden fixtures by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/nb PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``randqr`` from /root/reference/pkg/src (read-only; numba's cache is
redirected to /tmp so the reference tree is not written) and writes compressed
``.npz`` fixtures next to this script.  The GPU box never reads /root/reference;
tests consume only these committed fixtures.
"""

import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nb")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402
import randqr  # noqa: E402
from randqr.blocked import BlockConfig, block_qr, block_rrqr  # noqa: E402
from randqr.pivoting import SketchConfig  # noqa: E402
from randqr.rng import RngState, gaussian_matrix  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def composite_perm(f):
    """A[:, perm] = A P for permutation-pivot factorizations."""
    n = f.n
    perm = np.arange(n, dtype=np.int64)
    for t in f.p_transforms:
        order = t.op.order
        perm[t.offset: t.offset + len(order)] = perm[t.offset: t.offset + len(order)][order]
    return perm


# (tag, m, n, b, p, q, pivot_kind, rrqr, seed_a, seed_sketch)
SMALL = [
    ("m1_24x24_b6", 24, 24, 6, 0, 0, "permutation", False, 60, 61),
    ("m1_15x11_b4", 15, 11, 4, 0, 0, "permutation", False, 60, 61),
    ("m1_26x17_b5", 26, 17, 5, 0, 0, "permutation", False, 60, 61),
    ("m1_24x24_b6_p3", 24, 24, 6, 3, 0, "permutation", False, 62, 63),
    ("m1_q1_24x24_b6", 24, 24, 6, 0, 1, "permutation", False, 60, 61),
    ("m1_9x9_b9", 9, 9, 9, 0, 0, "permutation", False, 68, 69),
    ("m1_300x300_b50_p10", 300, 300, 50, 10, 0, "permutation", False, 0, 1),
    ("m1_200x130_b32_p2", 200, 130, 32, 2, 0, "permutation", False, 5, 6),
    ("m1_257x257_b64_p1", 257, 257, 64, 1, 0, "permutation", False, 7, 8),
    ("m2_24x24_b6", 24, 24, 6, 0, 0, "reflectors", False, 60, 61),
    ("m2_q2_24x24_b6_p2", 24, 24, 6, 2, 2, "reflectors", False, 60, 61),
    ("m2_160x160_b32_p8", 160, 160, 32, 8, 0, "reflectors", False, 3, 4),
    ("m3_24x24_b6_p2_q1", 24, 24, 6, 2, 1, "reflectors", True, 60, 61),
    ("m3_26x17_b5_p2_q1", 26, 17, 5, 2, 1, "reflectors", True, 60, 61),
    ("m3_300x300_b50_p25_q2", 300, 300, 50, 25, 2, "reflectors", True, 0, 1),
    ("m3_128x128_b32_p10_q1", 128, 128, 32, 10, 1, "reflectors", True, 9, 10),
]


def small_cases():
    out = {}
    for tag, m, n, b, p, q, kind, rr, sa, ss in SMALL:
        a = gaussian_matrix(m, n, RngState(sa))
        cfg = BlockConfig(b, SketchConfig(b, p, q), kind, rr)
        rng = RngState(ss)
        f = (block_rrqr if rr else block_qr)(a, cfg, rng)
        d = {"a": a, "r": f.r, "q": f.expand_q(), "p": f.expand_p(),
             "counter": np.int64(rng.counter), "cfg": np.array([m, n, b, p, q, int(kind == "reflectors"), int(rr), sa, ss])}
        if kind == "permutation" and not rr:
            d["perm"] = composite_perm(f)
        for k, v in d.items():
            out[f"{tag}/{k}"] = v
    np.savez_compressed(os.path.join(HERE, "small_factorizations.npz"), **out)


def rng_and_kernels():
    out = {}
    # stream pins: several seeds/counters, column-major, incl. a 64-bit seed
    for seed, counter, rows, cols in [(0, 0, 2, 2), (9000000000, 0, 3, 1), (1, 12345, 17, 5),
                                      (2**63 + 11, 7, 8, 8), (1, 0, 4096, 1)]:
        rng = RngState(seed, counter)
        out[f"rng/{seed}/{counter}/{rows}x{cols}"] = gaussian_matrix(rows, cols, rng)
    # raw integer words (for the bitwise integer-stream pin)
    from randqr.rng import _raw
    out["rng_words/seed1"] = _raw(1, np.arange(0, 1000, dtype=np.uint64))
    out["rng_words/seed_big"] = _raw(2**63 + 11, np.arange(0, 1000, dtype=np.uint64))
    # kernel-level pins: sweeps with and without pivoting, partial steps
    from randqr.householder import qr_column_pivoted, qr_unpivoted
    from randqr.pivoting import select_pivot_permutation, select_pivot_reflectors, build_sketch
    for tag, (m, n, s) in {"sq": (40, 40, 40), "tall": (300, 24, 24), "wide": (20, 90, 20), "part": (34, 500, 32)}.items():
        a = gaussian_matrix(m, n, RngState(100 + m))
        res = qr_column_pivoted(a, steps=s)
        out[f"cpqr/{tag}/a"] = a
        out[f"cpqr/{tag}/r"] = res.r
        out[f"cpqr/{tag}/perm"] = res.perm
        if m >= n:
            u = qr_unpivoted(a)
            out[f"qr/{tag}/r"] = u.r
            out[f"qr/{tag}/w"] = u.q.w
            out[f"qr/{tag}/y"] = u.q.y
    # ties and zero columns
    z = np.zeros((6, 5))
    z[:, 1] = 1.0
    z[:, 3] = 1.0  # equal norms: lowest index must win
    out["cpqr/ties/a"] = z
    out["cpqr/ties/perm"] = qr_column_pivoted(z).perm
    # pivot selection from a sketch
    x = gaussian_matrix(60, 50, RngState(200))
    y = build_sketch(x, SketchConfig(8, 4, 0), RngState(201))
    out["pivot/y"] = y
    out["pivot/order"] = select_pivot_permutation(y, 8).order
    rp = select_pivot_reflectors(y, 8)
    out["pivot/refl_w"] = rp.wy.w
    out["pivot/refl_y"] = rp.wy.y
    np.savez_compressed(os.path.join(HERE, "rng_kernels.npz"), **out)


def baseline_cfg1():
    """BASELINE cfg 1: 2000x2000 N(0,1) seed 0, b=64, p=10, sketch seed 1."""
    a = gaussian_matrix(2000, 2000, RngState(0))
    rng = RngState(1)
    f = block_qr(a, BlockConfig(64, SketchConfig(64, 10, 0)), rng)
    r = f.r
    out = {
        "perm": composite_perm(f),
        "diag": np.diag(r).copy(),
        "r_top": r[:64, :].copy(),
        "r_colnorm": np.linalg.norm(r, axis=0),
        "counter": np.int64(rng.counter),
        "a_checksum": np.array([a.sum(), np.abs(a).sum(), a[0, 0], a[-1, -1]]),
    }
    np.savez_compressed(os.path.join(HERE, "cfg1_n2000.npz"), **out)


def cfg2_small():
    """Scaled-down BASELINE cfg 2 (n=600): Haar U diag(10^(-8j/n)) V^T, b=64, p=10."""
    n = 600
    rng0 = RngState(0)
    u = randqr.haar_orthonormal(n, rng0)
    v = randqr.haar_orthonormal(n, rng0)
    s = 10.0 ** (-8.0 * np.arange(1, n + 1) / n)
    a = (u * s) @ v.T
    rng = RngState(1)
    f = block_qr(a, BlockConfig(64, SketchConfig(64, 10, 0)), rng)
    out = {"a": a, "perm": composite_perm(f), "r": f.r, "s": s, "counter": np.int64(rng.counter)}
    np.savez_compressed(os.path.join(HERE, "cfg2_n600.npz"), **out)
    # rank-revealing variant on a cfg-4-like spectrum (n=400, rank ~100)
    n = 400
    rng0 = RngState(0)
    u = randqr.haar_orthonormal(n, rng0)
    v = randqr.haar_orthonormal(n, rng0)
    s = np.maximum(10.0 ** (-12.0 * np.arange(1, n + 1) / 100), 1e-15)
    a = (u * s) @ v.T
    rng = RngState(1)
    f = block_rrqr(a, BlockConfig(32, SketchConfig(32, 10, 1), "reflectors", True), rng)
    out = {"a": a, "r": f.r, "s": s, "counter": np.int64(rng.counter)}
    np.savez_compressed(os.path.join(HERE, "cfg4_n400.npz"), **out)


if __name__ == "__main__":
    rng_and_kernels()
    small_cases()
    baseline_cfg1()
    cfg2_small()
    for fn in sorted(os.listdir(HERE)):
        if fn.endswith(".npz"):
            print(fn, os.path.getsize(os.path.join(HERE, fn)))
