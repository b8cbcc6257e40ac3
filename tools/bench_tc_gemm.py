"""Time the tcgen05 3xTF32 contraction at the C4 shapes (X: 20000 x 5000,
512 nodes): forward U = X Gamma (M=n, K=p) and transpose G = X^T [R|Z]
(M=p, K=n).  Prints per-call device time (split kernels included) and the
implied tensor throughput; run under ncu for the per-kernel split."""
import ctypes, sys
import torch
sys.path.insert(0, ".")
from paper_2502_09502_b200 import native

lib = native.lib()
def run(M, N, K, reps=10):
    A = torch.randn(M, K, device="cuda", dtype=torch.float32)
    B = torch.randn(N, K, device="cuda", dtype=torch.float32)
    ws = torch.empty(int(lib.l0_tc_gemm_workspace_bytes(M, N, K)), dtype=torch.uint8, device="cuda")
    C = torch.empty((64, N, M), dtype=torch.float32, device="cuda")
    so = ctypes.c_int32(0)
    call = lambda: native.check(lib.l0_tc_gemm_3xtf32(A.data_ptr(), 1, M, K, K, B.data_ptr(), 1, N, K,
                                   C.data_ptr(), M, 0, ctypes.byref(so), ws.data_ptr(), ws.numel(), None))
    for _ in range(2): call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): call()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    fl = 2.0 * M * N * K
    print(f"M={M} N={N} K={K} S={so.value}: {ms:.3f} ms/call  useful {fl/ms/1e9:.1f} TFLOP/s  "
          f"tensor(3x) {3*fl/ms/1e9:.1f} TFLOP/s", flush=True)
run(20000, 512, 5000)
run(5000, 512, 20000)
run(5000, 1024, 20000)
run(8192, 256, 8192)
