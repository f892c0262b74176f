"""One leaf QR launch pattern (m' x 16) for ncu source-level profiling."""
import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_1505_08115_b200 as rq
from paper_1505_08115_b200.errors import check
eng = rq.Engine()
mm = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
ld = mm + (mm & 1)
a0 = torch.randn(16, ld, dtype=torch.float64, device="cuda")
w = a0.clone(); v = torch.zeros_like(a0); t = torch.zeros(32, 32, dtype=torch.float64, device="cuda")
for _ in range(4):
    w.copy_(a0)
    check(eng.lib.rq_test_leaf_qr(eng.handle, ctypes.c_void_p(w.data_ptr()), ld, mm, 16,
                                  ctypes.c_void_p(v.data_ptr()), ld, ctypes.c_void_p(t.data_ptr()), 32))
torch.cuda.synchronize()
print("ok")
