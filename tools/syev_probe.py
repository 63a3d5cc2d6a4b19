"""Time bk_syev_d (n_need = d/3, as LOBPCG asks) for a range of d (tuning tool).
    BK_TRI_NO_PACKED=1 python tools/syev_probe.py 120 150 180 207"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2409_05572_b200 import load  # noqa: E402

f = load().lib
_D = C.c_void_p
f.bk_syev_work_bytes.restype = C.c_size_t
f.bk_syev_work_bytes.argtypes = [C.c_int]
f.bk_syev_d.argtypes = [C.c_int, _D, C.c_int, C.c_int, _D, _D, C.c_int, _D, _D, _D]
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
env = {k: v for k, v in os.environ.items() if k.startswith("BK_")}
for d in [int(a) for a in sys.argv[1:]] or [120, 150, 180, 207, 218, 288]:
    rng = np.random.default_rng(d)
    q, _ = np.linalg.qr(rng.standard_normal((d, d)))
    h = torch.as_tensor((q * np.linspace(0.01, 12, d)) @ q.T, device="cuda")
    vals = torch.zeros(d, dtype=torch.float64, device="cuda")
    z = torch.zeros((d, d), dtype=torch.float64, device="cuda")
    ws = torch.empty(f.bk_syev_work_bytes(d) // 8 + 1, dtype=torch.float64, device="cuda")
    info = torch.zeros(4, dtype=torch.int32, device="cuda")
    need = d if os.environ.get("PROBE_ALL") else d // 3  # SI / TraceMIN ask for all d pairs
    call = lambda: f.bk_syev_d(d, h.data_ptr(), d, need, vals.data_ptr(), z.data_ptr(), d, ws.data_ptr(),
                               info.data_ptr(), st)
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        call()
    e1.record()
    torch.cuda.synchronize()
    print(f"{env} d={d} n_need={need} {e0.elapsed_time(e1) / 10 * 1e3:8.1f} us")
