"""The experiment harness on the GPU against the reference's own CLI output.

tests/golden/cli_cells_n120.npz holds CSV cells written by the REFERENCE's ``randqr run``
(cli.py:45-58; made by tests/golden/make_golden_cli.py) at n = 120, b = 30, seed 1: cpqr, svd,
m1, m2, m3 on the fast / gauss / sshape matrices.  Here this library's CLI runs the same cells
(device matrix generators, the B200 factorizations, truncation errors read off R on the device)
and the tables must agree: same ranks, sigma_k, |R(k,k)| and spectral / Frobenius errors to
1e-9 relative (plus 1e-13 sigma_1 absolute for the errors that reach the rounding floor).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CELLS = ["fast_cpqr_q0", "fast_svd_q0", "fast_m1_q0", "fast_m2_q1", "fast_m3_q2", "gauss_m1_q0", "gauss_m3_q2",
         "sshape_m2_q0", "sshape_m3_q1_o10"]


def _parse(path):
    rows = open(path).read().strip().splitlines()
    assert rows[0] == "k,spectral_err,frobenius_err,r_diag,sigma"
    out = np.full((len(rows) - 1, 5), np.nan)
    for i, line in enumerate(rows[1:]):
        for j, f in enumerate(line.split(",")):
            if f != "":
                out[i, j] = float(f)
    return out


@pytest.mark.parametrize("tag", CELLS)
def test_cli_cell_matches_the_reference_csv(golden, tmp_path, tag):
    from paper_1505_08115_b200 import cli

    g = golden("cli_cells_n120.npz")
    n, b, seed = (int(x) for x in g["meta"])
    ref = g[tag]
    parts = tag.split("_")
    kind, method, q = parts[0], parts[1], int(parts[2][1:])
    argv = ["run", "--matrix", kind, "--n", str(n), "--block", str(b), "--method", method, "--q", str(q),
            "--seed", str(seed), "--out", str(tmp_path)]
    if len(parts) > 3:
        argv += ["--oversample", parts[3][1:]]
    assert cli.main(argv) == 0
    name = f"{kind}_{method}_q{q}.csv" if method in ("m2", "m3") else f"{kind}_{method}.csv"
    got = _parse(str(tmp_path / name))
    assert got.shape == ref.shape
    assert np.array_equal(np.isnan(got), np.isnan(ref)), "different ranks reported"
    s1 = ref[1, 4]
    for col, what in ((4, "sigma"), (3, "|R(k,k)|"), (1, "spectral"), (2, "frobenius")):
        ok = ~np.isnan(ref[:, col])
        d = np.abs(got[ok, col] - ref[ok, col])
        bound = 1e-9 * np.abs(ref[ok, col]) + 1e-13 * s1
        assert (d <= bound).all(), (what, float((d / np.maximum(bound, 1e-300)).max()))


def test_svd_baseline_is_the_svd(tmp_path):
    """svd = block_rrqr with one block of width n: R = diag(sigma), Q, P orthogonal, A P = Q R."""
    import paper_1505_08115_b200 as rq
    from paper_1505_08115_b200 import experiments as ex
    from paper_1505_08115_b200.matrices import MatrixSpec, gen_matrix

    a, sigma = gen_matrix(MatrixSpec("fast", 100, 3))
    f = ex.factorize(a, "svd", None, rq.RngState(5))
    r = f.r
    assert np.abs(r - np.diag(np.diag(r))).max() == 0.0
    assert np.allclose(np.diag(r), sigma, rtol=1e-10, atol=1e-14)
    q, p = f.expand_q(), f.expand_p()
    assert np.linalg.norm(a @ p - q @ r) <= 1e-13 * np.linalg.norm(a)
    assert np.linalg.norm(q.T @ q - np.eye(100)) <= 1e-12


def test_suite_writes_every_cell(tmp_path):
    from paper_1505_08115_b200 import cli

    assert cli.main(["suite", "--n", "48", "--block", "12", "--out", str(tmp_path)]) == 0
    names = sorted(p.name for p in tmp_path.iterdir())
    assert len(names) == 3 * (3 + 3 + 3), names
    assert "gauss_m3_q2.csv" in names and "sshape_svd.csv" in names
