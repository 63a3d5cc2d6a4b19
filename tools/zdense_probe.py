"""Time the complex Gram / symmetric Gram / update at config 5's shapes
(n = 2^20, widths 384 / 261, Rayleigh-Ritz d = 3 x width) through the bk_*_z
entry points, CUDA events, best of R.  BK_Z3M=0 selects the 4-product
real-view kernels, BK_ZGRAM / BK_ZGEMM the 3M tile variants.  Prints one JSON
line per shape: us, complex TFLOP/s (8 n a b; symmetric 4 n d (d+1))."""
import ctypes as C
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2409_05572_b200 import load  # noqa: E402

L = load().lib
_D, _I = C.c_void_p, C.c_int
L.bk_gram_z_work_bytes.restype = C.c_size_t
L.bk_gram_z_work_bytes.argtypes = [_I, _I, _I]
L.bk_gemm_z_work_bytes.restype = C.c_size_t
L.bk_gemm_z_work_bytes.argtypes = [_I, _I]
L.bk_gram_z.argtypes = [_I, _D, _I, _I, _D, _I, _I, _D, _I, _D, _D]
L.bk_gram_sym_z.argtypes = [_I, _D, _I, _D, _I, _I, _D, _I, _D, _D]
L.bk_gemm_z.argtypes = [_I, _D, _I, _I, _D, _I, _I, C.c_double, C.c_double, _D, _I, _D, _D]

n = int(os.environ.get("PROBE_N", 1 << 20))
R = int(os.environ.get("PROBE_R", 5))
tag = os.environ.get("PROBE_TAG", "")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
ld = 1152 + 8
S = torch.randn(n, 2 * ld, dtype=torch.float64, device="cuda")
AS = torch.randn(n, 2 * ld, dtype=torch.float64, device="cuda")
Y = torch.empty(n, 2 * 768, dtype=torch.float64, device="cuda")
Cm = torch.randn(1152, 2 * 768, dtype=torch.float64, device="cuda")
G = torch.empty(1152, 2 * 1152, dtype=torch.float64, device="cuda")
ws = torch.empty(L.bk_gram_z_work_bytes(n, 1152, 1152) // 8 + 1, dtype=torch.float64, device="cuda")
wg = torch.empty(L.bk_gemm_z_work_bytes(1152, 768) // 8 + 1, dtype=torch.float64, device="cuda")
p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731


def timeit(fn):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(R):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rc = fn()
        e1.record()
        torch.cuda.synchronize()
        assert rc == 0, rc
        best = min(best, e0.elapsed_time(e1) * 1e3)
    return best


def run(name, fn, flops):
    us = timeit(fn)
    print(json.dumps({"shape": name, "tag": tag, "n": n, "us": round(us, 1), "tflops": round(flops / us / 1e6, 2)}),
          flush=True)


for w in (384, 261):
    d = 3 * w
    run(f"gram_sym d={d}", lambda: L.bk_gram_sym_z(n, p(S), ld, p(AS), ld, d, p(G), d, p(ws), st), 4.0 * n * d * (d + 1))
    run(f"gram {2 * w}x{w}", lambda: L.bk_gram_z(n, p(S), ld, 2 * w, p(AS), ld, w, p(G), w, p(ws), st), 8.0 * n * 2 * w * w)
    run(f"gram {w}x{w}", lambda: L.bk_gram_z(n, p(S), ld, w, p(S), ld, w, p(G), w, p(ws), st), 8.0 * n * w * w)
    run(f"gemm {d}->{2 * w}", lambda: L.bk_gemm_z(n, p(S), ld, d, p(Cm), 2 * w, 2 * w, 1.0, 0.0, p(Y), 768, p(wg), st),
        8.0 * n * d * 2 * w)
    run(f"gemm {2 * w}->{w} beta=1", lambda: L.bk_gemm_z(n, p(S), ld, 2 * w, p(Cm), w, w, -1.0, 1.0, p(Y), 768, p(wg), st),
        8.0 * n * 2 * w * w)
    run(f"gemm {w}->{w}", lambda: L.bk_gemm_z(n, p(S), ld, w, p(Cm), w, w, 1.0, 0.0, p(Y), 768, p(wg), st),
        8.0 * n * w * w)
