import numpy as np, sys
for n in sys.argv[1:]:
    a = np.load(f"gpurun_out/la_off_{n}.npz"); b = np.load(f"gpurun_out/la_on_{n}.npz")
    same = np.array_equal(a["perm"], b["perm"])
    nd = np.argmax(a["perm"] != b["perm"]) if not same else -1
    print(n, "perm equal" if same else f"perm differs first at {nd}", "max rel diag diff", np.max(np.abs(a["d"] - b["d"]) / a["d"]))
