"""Golden CSV cells of the reference's experiment harness (randqr.cli "run", cli.py:45-58).

Run in the build container (where /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/nb PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_cli.py

Runs the REFERENCE's own CLI for a handful of cells at n = 120, b = 30 into a scratch directory
under /tmp, parses the CSVs and stores them as ``cli_cells_n120.npz`` next to this script (empty
CSV fields become NaN).  tests/test_gpu_experiments.py runs this library's CLI on the same cells.
"""

import os
import sys
import tempfile

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nb")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402
from randqr import cli  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
N, B, SEED = 120, 30, 1
# (kind, method, q, oversample)
CELLS = [
    ("fast", "cpqr", 0, None),
    ("fast", "svd", 0, None),
    ("fast", "m1", 0, None),
    ("fast", "m2", 1, None),
    ("fast", "m3", 2, None),
    ("gauss", "m1", 0, None),
    ("gauss", "m3", 2, None),
    ("sshape", "m2", 0, None),
    ("sshape", "m3", 1, 10),
]


def parse(path):
    rows = open(path).read().strip().splitlines()
    assert rows[0] == "k,spectral_err,frobenius_err,r_diag,sigma", rows[0]
    out = np.full((len(rows) - 1, 5), np.nan)
    for i, line in enumerate(rows[1:]):
        for j, field in enumerate(line.split(",")):
            if field != "":
                out[i, j] = float(field)
    return out


def main():
    fixtures = {}
    with tempfile.TemporaryDirectory(dir="/tmp") as tmp:
        for kind, method, q, over in CELLS:
            argv = ["run", "--matrix", kind, "--n", str(N), "--block", str(B), "--method", method, "--q", str(q),
                    "--seed", str(SEED), "--out", tmp]
            if over is not None:
                argv += ["--oversample", str(over)]
            assert cli.main(argv) == 0, argv
            name = f"{kind}_{method}_q{q}.csv" if method in ("m2", "m3") else f"{kind}_{method}.csv"
            tag = f"{kind}_{method}_q{q}" + (f"_o{over}" if over is not None else "")
            fixtures[tag] = parse(os.path.join(tmp, name))
    meta = np.array([N, B, SEED], dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "cli_cells_n120.npz"), meta=meta, **fixtures)
    print("wrote", sorted(fixtures))


if __name__ == "__main__":
    main()
