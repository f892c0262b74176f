"""Run single GEMM shapes through rq_test_gemm, one process per case (debug aid)."""
import subprocess
import sys

CASES = [(0, 64, 300, 300), (0, 256, 300, 1000), (0, 300, 60, 300), (1, 300, 300, 64), (1, 64, 300, 300),
         (1, 300, 60, 300), (0, 16, 8, 4)]

if len(sys.argv) > 1:
    import os
    sys.path.insert(0, os.getcwd())
    import numpy as np
    sys.argv = sys.argv[:1] + sys.argv[1:]
    mm, M, N, K = map(int, os.environ["CASE"].split(","))
    sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
    from test_gpu_kernels import _gemm
    from paper_1505_08115_b200 import Engine
    eng = Engine()
    rng = np.random.default_rng(0)
    A = rng.standard_normal((M, K) if mm else (K, M))
    B = rng.standard_normal((K, N))
    C = rng.standard_normal((M, N))
    out = _gemm(eng, mm, M, N, K, A, B, C, 1.0, 0.0)
    ref = (A if mm else A.T) @ B
    print("case", mm, M, N, K, "maxerr", np.abs(out - ref).max())
else:
    import os
    for c in CASES:
        env = dict(os.environ, CASE=",".join(map(str, c)))
        r = subprocess.run([sys.executable, __file__, "run"], env=env, capture_output=True, text=True, timeout=120)
        print(c, "rc", r.returncode, (r.stdout.strip().splitlines() or [""])[-1], (r.stderr.strip().splitlines() or [""])[-1][:200])
