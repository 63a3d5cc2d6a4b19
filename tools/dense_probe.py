"""Time the config-2 Gram / update shapes through the C ABI (tuning tool).
    BK_NARROW=2 python tools/dense_probe.py [n]
Prints one line per shape: TF/s (algorithmic flops / CUDA-event time, 20 calls)."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2409_05572_b200 import load  # noqa: E402

f = load().lib
_D = C.c_void_p
f.bk_gram_work_bytes.restype = C.c_size_t
f.bk_gram_work_bytes.argtypes = [C.c_int, C.c_int, C.c_int]
f.bk_gram_d.argtypes = [C.c_int, _D, C.c_int, C.c_int, _D, C.c_int, C.c_int, _D, C.c_int, _D, _D]
f.bk_gram_sym_d.argtypes = [C.c_int, _D, C.c_int, _D, C.c_int, C.c_int, _D, C.c_int, _D, _D]
f.bk_gemm_d.argtypes = [C.c_int, _D, C.c_int, C.c_int, _D, C.c_int, C.c_int, C.c_double, C.c_double, _D, C.c_int, _D]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
ld = 296
x = torch.randn(n, ld, dtype=torch.float64, device="cuda")
y = torch.randn(n, ld, dtype=torch.float64, device="cuda")
c = torch.randn(ld, ld, dtype=torch.float64, device="cuda")
ws = torch.empty(f.bk_gram_work_bytes(n, 288, 288) // 8 + 1, dtype=torch.float64, device="cuda")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)


def timeit(call, flops):
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
    return ms * 1e3, flops / (ms * 1e-3) / 1e12


out = {}
for a, b in [(138, 69), (192, 96), (96, 96)]:
    us, tf = timeit(lambda: f.bk_gram_d(n, x.data_ptr(), ld, a, y.data_ptr(), ld, b, c.data_ptr(), ld,
                                        ws.data_ptr(), st), 2.0 * n * a * b)
    out[f"gram {a}x{b}"] = (us, tf)
for d, same in [(207, False), (288, False), (69, True), (96, True)]:
    yy = x if same else y
    us, tf = timeit(lambda: f.bk_gram_sym_d(n, x.data_ptr(), ld, yy.data_ptr(), ld, d, c.data_ptr(), ld,
                                            ws.data_ptr(), st), 1.0 * n * d * (d + 1))
    out[f"gram_sym {d}{' (X=Y)' if same else ''}"] = (us, tf)
for d, k, beta in [(207, 138, 0.0), (138, 69, 1.0), (69, 69, 0.0), (288, 192, 0.0), (192, 96, 1.0), (96, 96, 0.0)]:
    us, tf = timeit(lambda: f.bk_gemm_d(n, x.data_ptr(), ld, d, c.data_ptr(), ld, k, 1.0, beta, y.data_ptr(), ld,
                                        st), 2.0 * n * d * k)
    out[f"gemm {d}->{k} beta={beta:g}"] = (us, tf)
env = {k: v for k, v in os.environ.items() if k.startswith("BK_")}
for k, (us, tf) in out.items():
    print(f"{json.dumps(env)} {k:28s} {us:9.1f} us {tf:6.2f} TF/s")
