"""Time / profile one bk_gram_d shape on the B200 (tuning tool).
    python tools/gram_probe.py A B [n]"""
import ctypes as C
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2409_05572_b200 import load  # noqa: E402

f = load().lib
_D = C.c_void_p
f.bk_gram_work_bytes.restype = C.c_size_t
f.bk_gram_work_bytes.argtypes = [C.c_int, C.c_int, C.c_int]
f.bk_gram_d.argtypes = [C.c_int, _D, C.c_int, C.c_int, _D, C.c_int, C.c_int, _D, C.c_int, _D, _D]
a, b = int(sys.argv[1]), int(sys.argv[2])
n = int(sys.argv[3]) if len(sys.argv) > 3 else 262144
ld = max(344, (max(a, b) + 7) // 8 * 8)
x = torch.randn(n, ld, dtype=torch.float64, device="cuda")
y = torch.randn(n, ld, dtype=torch.float64, device="cuda")
c = torch.zeros(a, b, dtype=torch.float64, device="cuda")
ws = torch.empty(f.bk_gram_work_bytes(n, a, b) // 8 + 1, dtype=torch.float64, device="cuda")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
call = lambda: f.bk_gram_d(n, x.data_ptr(), ld, a, y.data_ptr(), ld, b, c.data_ptr(), b, ws.data_ptr(), st)
for _ in range(3):
    call()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    call()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(f"gram {a}x{b} n={n}: {ms:.4f} ms {2 * n * a * b / ms / 1e9:.2f} TFLOP/s")
