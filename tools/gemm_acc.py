import ctypes, sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_1505_08115_b200 as rq
from paper_1505_08115_b200.errors import check
eng = rq.Engine()
torch.backends.cuda.matmul.allow_tf32 = False
for (M, N, K) in [(512, 512, 256), (512, 512, 4096)]:
    rng = np.random.default_rng(0)
    A = rng.standard_normal((K, M)).astype(np.float32)   # TN: A stored K x M
    B = rng.standard_normal((K, N)).astype(np.float32)
    at = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()  # storage (M, K): column-major K x M
    bt = torch.from_numpy(np.ascontiguousarray(B.T)).cuda()
    ct = torch.zeros((N, M), dtype=torch.float32, device="cuda")
    check(eng.lib.rq_gemm_f32(eng.handle, 0, M, N, K, ctypes.c_void_p(at.data_ptr()), K, K, M, 0, 0,
                              ctypes.c_void_p(bt.data_ptr()), K, K, N, 0, 0, ctypes.c_void_p(ct.data_ptr()), M, 1.0, 0.0))
    ours = ct.cpu().numpy().T.astype(np.float64)
    ref = A.T.astype(np.float64) @ B.astype(np.float64)
    sg = (torch.from_numpy(A.T).cuda() @ torch.from_numpy(B).cuda()).cpu().numpy().astype(np.float64)
    scale = np.abs(A.T.astype(np.float64)) @ np.abs(B.astype(np.float64))
    for name, x in (("tf32x3", ours), ("sgemm", sg)):
        e = np.abs(x - ref) / scale
        print(M, N, K, name, "max", e.max(), "rms", np.sqrt((e**2).mean()), "abs/rms", np.abs(x-ref).max()/np.sqrt((ref**2).mean()))

# throughput at the trailing-update shapes (3 tensor-core products per k; the 2MNK count)
for (mm, M, N, K) in [(1, 10000, 10000, 256), (0, 256, 10000, 10000)]:
    a_rows, a_cols = (M, K) if mm else (K, M)
    at = torch.randn((a_cols, a_rows), dtype=torch.float32, device="cuda")
    bt = torch.randn((N, K), dtype=torch.float32, device="cuda")
    ct = torch.zeros((N, M), dtype=torch.float32, device="cuda")
    def run():
        check(eng.lib.rq_gemm_f32(eng.handle, mm, M, N, K, ctypes.c_void_p(at.data_ptr()), a_rows, a_rows, a_cols, 0, 0,
                                  ctypes.c_void_p(bt.data_ptr()), K, K, N, 0, 0, ctypes.c_void_p(ct.data_ptr()), M,
                                  -1.0, 1.0))
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{'NN' if mm else 'TN'} {M}x{N}x{K}: {ms:.3f} ms, {2*M*N*K/ms/1e9:.1f} TFLOP/s (2MNK), "
          f"C traffic {(2 if mm else 1)*4*M*N/ms/1e6:.0f} GB/s")
