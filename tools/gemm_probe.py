"""Time one bk_gemm_d shape on the B200 (tuning tool).
    python tools/gemm_probe.py D K [n]     # Y (n x K) = X (n x D) C (D x K)"""
import ctypes as C
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2409_05572_b200 import load  # noqa: E402

f = load().lib
_D = C.c_void_p
f.bk_gemm_d.argtypes = [C.c_int, _D, C.c_int, C.c_int, _D, C.c_int, C.c_int, C.c_double, C.c_double, _D, C.c_int, _D]
d, k = int(sys.argv[1]), int(sys.argv[2])
n = int(sys.argv[3]) if len(sys.argv) > 3 else 262144
ld = (max(d, k) + 7) // 8 * 8
x = torch.randn(n, ld, dtype=torch.float64, device="cuda")
cm = torch.randn(d, k, dtype=torch.float64, device="cuda")
y = torch.zeros(n, ld, dtype=torch.float64, device="cuda")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
call = lambda: f.bk_gemm_d(n, x.data_ptr(), ld, d, cm.data_ptr(), k, k, 1.0, 0.0, y.data_ptr(), ld, st)
for _ in range(3):
    call()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    call()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"gemm {d}x{k} n={n}: {ms:.4f} ms {2 * n * d * k / ms / 1e9:.2f} TFLOP/s")
