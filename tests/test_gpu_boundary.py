"""Drop-in boundary semantics on the GPU (round 2):

* each Factorization owns its factors (blocked.py:122-149) even when two share an Engine;
* per-panel ``q_transforms`` / ``p_transforms`` proxies multiply out to expand_q / expand_p
  (QTransform.left_multiply / RightTransform.right_multiply, blocked.py:77-119);
* the HQRRP downdate identity (SURVEY section 8 "Two sketch modes"), checked independently of
  the driver's evaluation order: after every panel the device's downdated sketch equals
  (G Q)[:, s:] A22' and, equivalently, (G A P)[:, s:] - (G A P)[:, :s] R11^{-1} R12;
* error paths of rq_factorize_host and the RNG counter after a sketch-width error.
"""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rq():
    import paper_1505_08115_b200 as m

    return m


def _cfg(rq, b, p, q=0, refl=False, rr=False):
    return rq.BlockConfig(b, rq.SketchConfig(b, p, q), "reflectors" if refl else "permutation", rr)


def _check(a, f, tol=1e-13):
    m, n = a.shape
    q = f.expand_q()
    p = f.expand_p()
    scale = np.linalg.norm(a)
    assert np.linalg.norm(a @ p - q @ f.r[:n, :]) <= tol * scale
    assert np.linalg.norm(q.T @ q - np.eye(n)) <= tol * np.sqrt(m)


@pytest.mark.parametrize("kind", ["m1", "m1_downdate", "m2", "m3"])
def test_two_factorizations_share_an_engine(rq, kind):
    """f1's factors survive f2 on the same Engine (same shapes: the old failure was silent)."""
    rng = np.random.default_rng(11)
    a1 = np.asfortranarray(rng.standard_normal((300, 260)))
    a2 = np.asfortranarray(rng.standard_normal((300, 260)))
    eng = rq.Engine()
    kw = {"engine": eng}
    if kind == "m1_downdate":
        kw["sketch"] = "downdate"
    if kind == "m3":
        call, cfg = rq.block_rrqr, _cfg(rq, 40, 8, 1, refl=True, rr=True)
    else:
        call, cfg = rq.block_qr, _cfg(rq, 40, 8, 0, refl=(kind == "m2"))
    f1 = call(a1, cfg, rq.RngState(3), **kw)
    f2 = call(a2, cfg, rq.RngState(3), **kw)
    f3 = call(a1, cfg, rq.RngState(4), **kw)
    _check(a1, f1, 1e-12)
    _check(a2, f2, 1e-12)
    _check(a1, f3, 1e-12)
    q1 = f1.expand_q()
    del f3
    f4 = call(a2, cfg, rq.RngState(5), **kw)
    assert np.array_equal(f1.expand_q(), q1)
    _check(a2, f4, 1e-12)


def test_q_transforms_multiply_out_to_q(rq):
    a = np.asfortranarray(np.random.default_rng(2).standard_normal((330, 300)))
    f = rq.block_qr(a, _cfg(rq, 64, 6), rq.RngState(1))
    qt = f.q_transforms
    assert [t.offset for t in qt] == list(range(0, 300, 64))
    x = np.eye(330, 300)
    for t in reversed(qt):
        x = t.left_multiply(x)
    q = f.expand_q()
    assert np.abs(x - q).max() <= 1e-13
    y = np.random.default_rng(3).standard_normal((330, 5))
    qfull = f.expand_q(330)
    assert np.abs(f.apply_q(y, transpose=True) - qfull.T @ y).max() <= 1e-12
    assert np.abs(f.apply_q(y) - qfull @ y).max() <= 1e-12
    z = y.copy()
    for t in qt:
        z = t.left_multiply_transposed(z)
    assert np.abs(z - qfull.T @ y).max() <= 1e-12


def test_p_transforms_multiply_out_to_p(rq, golden):
    from oracle import randqr_oracle as O

    a = O.gaussian_matrix(300, 300, O.RngState(0))
    f = rq.block_qr(a, _cfg(rq, 50, 10), rq.RngState(1))
    p = np.eye(300)
    for t in f.p_transforms:
        p = t.right_multiply(p)
    assert np.array_equal(p, f.expand_p())
    # reflector pivots and block_rrqr: orthogonal right factors on the device
    g = golden("small_factorizations.npz")
    for tag, rr in (("m2_160x160_b32_p8", False), ("m3_128x128_b32_p10_q1", True)):
        m, n, b, pp, q, refl, _, sa, ss = (int(x) for x in g[f"{tag}/cfg"])
        call = rq.block_rrqr if rr else rq.block_qr
        f = call(g[f"{tag}/a"], _cfg(rq, b, pp, q, refl=True, rr=rr), rq.RngState(ss))
        p = np.eye(n)
        for t in f.p_transforms:
            p = t.right_multiply(p)
        assert np.abs(p - f.expand_p()).max() <= 1e-13
        assert np.abs(p - g[f"{tag}/p"]).max() <= 1e-10


@pytest.mark.parametrize("m,n,b,p", [(600, 500, 64, 8), (420, 420, 50, 10)])
def test_downdate_identity_after_every_panel(rq, m, n, b, p):
    """Y2,downdated == (G Q)[:, s:] A22' to 1e-13 relative after each panel (SURVEY section 8,
    measured there at 6.5e-16 with the reference's own kernels)."""
    from oracle import randqr_oracle as O
    from paper_1505_08115_b200.errors import check

    wdt = b + p
    a = O.gaussian_matrix(m, n, O.RngState(17))
    g = O.gaussian_matrix(m, wdt, O.RngState(5)).T  # G = Omega^T, drawn first in downdate mode
    eng = rq.Engine()
    recs = []

    def insp(panel, w):
        s = panel * b
        if s >= n:
            return
        y = np.zeros((wdt, n - s), order="F")
        perm = np.zeros(n, dtype=np.int64)
        check(eng.lib.rq_snapshot_sketch(eng.handle, y.ctypes.data_as(ctypes.c_void_p), wdt,
                                         perm.ctypes.data_as(ctypes.c_void_p)))
        recs.append((panel, s, w.copy(), y, perm))

    f = rq.block_qr(a, _cfg(rq, b, p), rq.RngState(5), insp, engine=eng, sketch="downdate")
    assert len(recs) == (n - 1) // b
    ga = g @ a
    for panel, s, w, y, perm in recs:
        gap = ga[:, perm]
        r11, r12 = np.triu(w[:s, :s]), w[:s, s:]
        expect = gap[:, s:] - gap[:, :s] @ np.linalg.solve(r11, r12)
        assert np.linalg.norm(y - expect) <= 1e-13 * np.linalg.norm(y), panel
        # the survey's form: (G Q_i)[:, s:] A22', Q_i = U_1 ... U_i from the q_transforms proxies
        qi = f._apply_q(0, panel, False, np.eye(m))
        expect2 = (g @ qi)[:, s:] @ w[s:, s:]
        assert np.linalg.norm(y - expect2) <= 1e-13 * np.linalg.norm(y), panel
    assert np.array_equal(recs[-1][4][: recs[-1][1]], f.perm[: recs[-1][1]])


def test_downdate_sketch_width_error_counter_matches_oracle(rq):
    from oracle import randqr_oracle as O

    a = O.gaussian_matrix(90, 70, O.RngState(2))
    cfg = _cfg(rq, 32, 8)
    rng = rq.RngState(6)
    ref_rng = O.RngState(6)
    with pytest.raises(ValueError):
        rq.block_qr(a, cfg, rng, sketch="downdate")
    with pytest.raises(ValueError):
        O.block_qr_downdate(a, O.BlockConfig(32, O.SketchConfig(32, 8, 0)), ref_rng)
    assert rng.counter == ref_rng.counter == 90 * 40


def test_factorize_host_rejects_short_leading_dimensions(rq):
    from paper_1505_08115_b200 import _lib

    m, n = 64, 48
    a = np.asfortranarray(np.random.default_rng(0).standard_normal((m, n)))
    eng = rq.Engine()
    cfg = _lib.rq_config(16, 4, 0, -1, _lib.RQ_PIVOT_PERMUTATION, 0, _lib.RQ_SKETCH_FRESH, 0)
    hr = np.zeros((m, n), order="F")
    ctr = ctypes.c_uint64(0)
    rc = eng.lib.rq_factorize_host(eng.handle, ctypes.byref(cfg), m, n, a.ctypes.data_as(ctypes.c_void_p), m,
                                   ctypes.c_uint64(1), ctypes.byref(ctr), hr.ctypes.data_as(ctypes.c_void_p), m - 1,
                                   None)
    assert rc == _lib.RQ_EVALUE and b"ldr" in eng.lib.rq_last_error()
    rc = eng.lib.rq_factorize_host(eng.handle, ctypes.byref(cfg), m, n, a.ctypes.data_as(ctypes.c_void_p), m - 2,
                                   ctypes.c_uint64(1), ctypes.byref(ctr), hr.ctypes.data_as(ctypes.c_void_p), m, None)
    assert rc == _lib.RQ_EVALUE
    assert ctr.value == 0
    # a valid call on the same context still works and equals the device path
    rc = eng.lib.rq_factorize_host(eng.handle, ctypes.byref(cfg), m, n, a.ctypes.data_as(ctypes.c_void_p), m,
                                   ctypes.c_uint64(1), ctypes.byref(ctr), hr.ctypes.data_as(ctypes.c_void_p), m, None)
    assert rc == _lib.RQ_OK
    f = rq.block_qr(a, _cfg(rq, 16, 4), rq.RngState(1))
    assert np.array_equal(np.triu(hr), f.r)


def test_fresh_engine_after_free_keeps_pivots(rq):
    """A new context reusing freed device memory (same addresses) must not read stale sketch
    exchange words: many engine-per-call factorizations give identical pivots."""
    from oracle import randqr_oracle as O

    a = O.gaussian_matrix(2000, 2000, O.RngState(0))
    perms = []
    for _ in range(4):
        eng = rq.Engine()
        f = rq.block_qr(a, _cfg(rq, 64, 10), rq.RngState(1), engine=eng)
        perms.append(f.perm.copy())
        del f
        eng.close()
    for p in perms[1:]:
        assert np.array_equal(p, perms[0])
