"""CPU checks of the experiment harness mirror (paper_1505_08115_b200.experiments / cli, the
reference's experiments.py / cli.py): method defaults, cell names, the CSV layout against the
reference's own CSVs (tests/golden/cli_cells_n120.npz, made by tests/golden/make_golden_cli.py),
and the CLI's argument errors (exit code 2, no GPU work)."""

import numpy as np
import pytest


def test_method_config_defaults():
    from paper_1505_08115_b200 import experiments as ex

    assert ex.method_config("cpqr", 50) is None and ex.method_config("svd", 50) is None
    c1 = ex.method_config("m1", 50)
    assert (c1.block, c1.sketch.width, c1.sketch.oversample, c1.sketch.power, c1.pivot_kind, c1.rrqr) \
        == (50, 50, 0, 0, "permutation", False)
    c2 = ex.method_config("m2", 40, 2)
    assert (c2.sketch.oversample, c2.sketch.power, c2.pivot_kind, c2.rrqr) == (0, 2, "reflectors", False)
    c3 = ex.method_config("m3", 50, 1)
    assert (c3.sketch.oversample, c3.sketch.power, c3.rrqr) == (25, 1, True)
    assert ex.method_config("m3", 50, 1, 7).sketch.oversample == 7
    with pytest.raises(ValueError):
        ex.method_config("lu", 50)


def test_cell_filenames():
    from paper_1505_08115_b200 import experiments as ex

    assert ex.cell_filename("fast", "m3", 2) == "fast_m3_q2.csv"
    assert ex.cell_filename("gauss", "m2", 0) == "gauss_m2_q0.csv"
    assert ex.cell_filename("sshape", "cpqr", 0) == "sshape_cpqr.csv"
    assert ex.cell_filename("fast", "svd", 1) == "fast_svd.csv"


def _parse(path):
    rows = open(path).read().strip().splitlines()
    out = np.full((len(rows) - 1, 5), np.nan)
    for i, line in enumerate(rows[1:]):
        for j, f in enumerate(line.split(",")):
            if f != "":
                out[i, j] = float(f)
    return rows[0], out


def test_write_csv_reproduces_the_reference_layout(golden, tmp_path):
    """Feeding the reference's own numbers through write_csv gives back the same table
    (header, a row per k = 0..n, empty fields where undefined, 17 significant digits)."""
    from paper_1505_08115_b200 import experiments as ex
    from paper_1505_08115_b200.metrics import DiagComparison, ErrorCurve

    g = golden("cli_cells_n120.npz")
    n, b, _ = (int(x) for x in g["meta"])
    ref = g["fast_m3_q2"]
    ks = [int(k) for k in ref[:, 0] if not np.isnan(ref[int(k), 1])]
    assert ks == list(range(0, n, b)) + [n]
    curve = ErrorCurve(ks, [ref[k, 1] for k in ks], [ref[k, 2] for k in ks], "m3")
    diag = DiagComparison(ref[1:, 3].copy(), ref[1:, 4].copy())
    path = tmp_path / "c.csv"
    ex.write_csv(str(path), curve, diag)
    hdr, got = _parse(str(path))
    assert hdr == "k,spectral_err,frobenius_err,r_diag,sigma"
    assert got.shape == ref.shape
    assert np.array_equal(np.isnan(got), np.isnan(ref))
    assert np.array_equal(got[~np.isnan(got)], ref[~np.isnan(ref)])


def test_cli_argument_errors_exit_2(tmp_path):
    from paper_1505_08115_b200 import cli

    assert cli.main(["run", "--matrix", "fast", "--method", "m3", "--oversample", "-1", "--out", str(tmp_path)]) == 2
    with pytest.raises(SystemExit) as e:
        cli.main(["run", "--matrix", "nope", "--method", "m3", "--out", str(tmp_path)])
    assert e.value.code == 2
    with pytest.raises(SystemExit) as e:
        cli.main(["run", "--matrix", "fast", "--method", "m3", "--q", "3", "--out", str(tmp_path)])
    assert e.value.code == 2
