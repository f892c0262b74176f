"""Per-panel phase breakdown of one HQRRP factorization (tuning aid; run on the GPU box).

    RQ_PHASES=2 python tools/phase_seq.py N [N ...]

Runs a warm-up and one measured downdated-sketch factorization per n and prints, per panel, the
main-stream time between the phase events of Ctx::factorize_perm (driver.cu).
"""
import ctypes
import os
import subprocess
import sys

NAMES = {1: "panel_qr", 2: "cpqr||W", 3: "wait_WT", 4: "W2,top", 5: "downdate", 6: "sketch", 7: "moves",
         8: "final", 10: "trail", 11: "small_q", 12: "R,moves"}

if os.environ.get("_RQ_CHILD") != "1":
    for n in sys.argv[1:] or ["10000"]:
        env = dict(os.environ, RQ_PHASES="2", _RQ_CHILD="1")
        r = subprocess.run([sys.executable, __file__, n], env=env, capture_output=True, text=True)
        lines = [ln for ln in r.stderr.splitlines() if ln.startswith("[rq phase-seq]")]
        hlines = [ln for ln in r.stderr.splitlines() if ln.startswith("[rq phase-host]")]
        if not lines:
            print(r.stdout, r.stderr[-3000:])
            continue
        seq = [(int(t.split(":")[0]), float(t.split(":")[1])) for t in lines[-1].split()[2:]]
        panels, cur = [], {}
        for pid, ms in seq:
            if pid == 1 and cur:
                panels.append(cur)
                cur = {}
            cur[pid] = cur.get(pid, 0.0) + ms
        panels.append(cur)
        cols = [1, 2, 11, 12, 3, 4, 5, 6, 7, 8]
        print(f"n={n}: total {sum(ms for _, ms in seq):.2f} ms, {len(panels)} panels")
        print("panel " + " ".join(f"{NAMES[c]:>9s}" for c in cols) + "     sum")
        tot = {c: 0.0 for c in cols}
        for i, p in enumerate(panels):
            for c in cols:
                tot[c] += p.get(c, 0.0)
            if i < 6 or i % 8 == 0 or i >= len(panels) - 3:
                print(f"{i:5d} " + " ".join(f"{p.get(c, 0.0):9.3f}" for c in cols) + f" {sum(p.values()):7.3f}")
        print("total " + " ".join(f"{tot[c]:9.2f}" for c in cols))
        if hlines:  # host enqueue time per panel vs device time per panel
            hseq = [(int(t.split(":")[0]), float(t.split(":")[1])) for t in hlines[-1].split()[2:]]
            hp, cur = [], 0.0
            first = True
            for pid, ms in hseq:
                if pid == 1 and not first:
                    hp.append(cur)
                    cur = 0.0
                first = False
                cur += ms
            hp.append(cur)
            print("host enqueue ms per panel (vs device):")
            for i, (p, h) in enumerate(zip(panels, hp)):
                if i < 4 or i % 8 == 0 or i >= len(panels) - 3:
                    print(f"  panel {i:3d}: host {h:7.3f}  device {sum(p.values()):7.3f}")
            print(f"  total host {sum(hp):.2f} ms, device {sum(ms for _, ms in seq):.2f} ms")
    sys.exit(0)

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_1505_08115_b200 as rq  # noqa: E402
from paper_1505_08115_b200 import _lib  # noqa: E402
from paper_1505_08115_b200.errors import check  # noqa: E402

n = int(sys.argv[1])
b, p = 256, 16
# RQ_NEWSTREAM=1: the library's main stream is a created (non-default) stream, as in bench.py
eng = rq.Engine(0, stream=torch.cuda.Stream()) if os.environ.get("RQ_NEWSTREAM") == "1" else rq.Engine()
torch.cuda.set_stream(eng.stream)
a0, ld = rq.gaussian_matrix_device(n, n, rq.RngState(0), engine=eng)
work = torch.empty_like(a0)
perm = torch.empty(n, dtype=torch.int64, device=a0.device)
cfg = _lib.rq_config(b, p, 0, -1, _lib.RQ_PIVOT_PERMUTATION, 0, _lib.RQ_SKETCH_DOWNDATE, 0)
for _ in range(2):
    work.copy_(a0)
    ctr = ctypes.c_uint64(0)
    check(eng.lib.rq_factorize(eng.handle, ctypes.byref(cfg), n, n, ctypes.c_void_p(work.data_ptr()), ld,
                               ctypes.c_uint64(1), ctypes.byref(ctr), ctypes.c_void_p(perm.data_ptr())))
    torch.cuda.synchronize()
