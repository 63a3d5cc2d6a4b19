"""K1w (window-staged SpMM) probe: plan statistics on the host, and with --gpu the
kernel's time against the plain K1 on the same matrix (CUDA events, L2 flushed
between calls) plus a bit-identity check.

    python tools/spmm_win_probe.py --config 2 --tiles 64,128,256            # host only
    python tools/spmm_win_probe.py --config 2 --tiles 128 --gpu --ks 69,96,138
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2409_05572_b200 import LIB_PATH  # noqa: E402
from paper_2409_05572_b200 import workloads as W  # noqa: E402


def plan(lib, n, frp, fcol, fval, tile, wcap):
    lib.bk_spmm_win_plan.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
    lib.bk_spmm_win_plan_info.argtypes = [C.c_void_p] + [C.POINTER(C.c_int)] * 5 + [C.POINTER(C.c_double)]
    lib.bk_spmm_win_plan_arrays.argtypes = [C.c_void_p] + [C.POINTER(C.c_void_p)] * 5 + [C.POINTER(C.c_int64)]
    lib.bk_spmm_win_plan_free.argtypes = [C.c_void_p]
    h = C.c_void_p()
    rc = lib.bk_spmm_win_plan(n, frp.ctypes.data, fcol.ctypes.data, fval.ctypes.data, tile, wcap, C.byref(h))
    assert rc == 0, rc
    ok, t, nt, wmax, nzmax = (C.c_int() for _ in range(5))
    lpr = C.c_double()
    lib.bk_spmm_win_plan_info(h, ok, t, nt, wmax, nzmax, lpr)
    ptrs = [C.c_void_p() for _ in range(5)]
    wl = C.c_int64()
    lib.bk_spmm_win_plan_arrays(h, *[C.byref(p) for p in ptrs], C.byref(wl))
    nnz = int(frp[-1])

    def arr(p, ctype, count, dt):
        return np.ctypeslib.as_array(C.cast(p, C.POINTER(ctype)), shape=(count,)).astype(dt, copy=True)
    out = dict(ok=ok.value, tile=t.value, ntiles=nt.value, wmax=wmax.value, nzmax=nzmax.value,
               loads_per_row=lpr.value,
               rp2=arr(ptrs[0], C.c_int32, n + 1, np.int32), code=arr(ptrs[1], C.c_int32, nnz, np.int32),
               val2=arr(ptrs[2], C.c_double, nnz, np.float64), wptr=arr(ptrs[3], C.c_int32, nt.value + 1, np.int32),
               wrow=arr(ptrs[4], C.c_int32, wl.value, np.int32))
    lib.bk_spmm_win_plan_free(h)
    return out


def matrix(cfg, side):
    if cfg == "2":
        rp, col, val = W.grid_laplacian((side or 64,) * 3)
        n = (side or 64) ** 3
    elif cfg == "4":
        w = W.config4(side=side or 96, x0=False)
        rp, col, val, n = w.row_ptr, w.col, w.val, w.n
    elif cfg == "1":
        rp, col, val = W.grid_laplacian((side or 100,) * 2)
        n = (side or 100) ** 2
    else:
        raise SystemExit("config 1, 2 or 4")
    full = W.full_from_lower(n, rp, col, val)
    return n, full.indptr.astype(np.int32), full.indices.astype(np.int32), np.ascontiguousarray(full.data)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="2")
    ap.add_argument("--side", type=int, default=0)
    ap.add_argument("--tiles", default="64,128,256")
    ap.add_argument("--wcap", type=int, default=1 << 20)
    ap.add_argument("--gpu", action="store_true")
    ap.add_argument("--ks", default="69,96,138")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    lib = C.CDLL(LIB_PATH)
    n, frp, fcol, fval = matrix(a.config, a.side)
    nnz = int(frp[-1])
    for tile in map(int, a.tiles.split(",")):
        t0 = time.time()
        p = plan(lib, n, frp, fcol, fval, tile, a.wcap)
        sz = np.diff(p["wptr"])
        info = dict(config=a.config, n=n, nnz=nnz, tile=p["tile"], ok=p["ok"], ntiles=p["ntiles"], wmax=p["wmax"],
                    w_mean=float(sz.mean()), w_p99=float(np.percentile(sz, 99)), nzmax=p["nzmax"],
                    loads_per_row=round(p["loads_per_row"], 3), nnz_per_row=round(nnz / n, 2),
                    plan_seconds=round(time.time() - t0, 2))
        print(json.dumps(info), flush=True)
        if not a.gpu:
            continue
        import torch
        D = C.c_void_p
        lib.bk_spmm_d.argtypes = [C.c_int, D, D, D, D, C.c_int, C.c_int, D, C.c_int, D]
        lib.bk_spmm_win_d.argtypes = [C.c_int] * 5 + [D] * 5 + [D, C.c_int, C.c_int, D, C.c_int, D]
        dev = lambda v: torch.from_numpy(np.ascontiguousarray(v)).cuda()
        d = {k: dev(p[k]) for k in ("rp2", "code", "val2", "wptr", "wrow")}
        t_rp, t_c, t_v = dev(frp), dev(fcol), dev(fval)
        flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        st = torch.cuda.current_stream().cuda_stream
        for k in map(int, a.ks.split(",")):
            ld = (k + 7) // 8 * 8
            x = torch.randn(n, ld, dtype=torch.float64, device="cuda")
            y1, y2 = torch.zeros_like(x), torch.zeros_like(x)

            def plain():
                return lib.bk_spmm_d(n, t_rp.data_ptr(), t_c.data_ptr(), t_v.data_ptr(), x.data_ptr(), ld, k,
                                     y1.data_ptr(), ld, st)

            def win():
                return lib.bk_spmm_win_d(n, p["tile"], p["ntiles"], p["wmax"], p["nzmax"], d["rp2"].data_ptr(),
                                         d["code"].data_ptr(), d["val2"].data_ptr(), d["wptr"].data_ptr(),
                                         d["wrow"].data_ptr(), x.data_ptr(), ld, k, y2.data_ptr(), ld, st)
            res = {}
            for name, f in (("plain", plain), ("win", win)):
                ts = []
                for r in range(a.reps + 3):
                    flush.zero_()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    rc = f()
                    e1.record()
                    torch.cuda.synchronize()
                    assert rc == 0, (name, rc)
                    if r >= 3:
                        ts.append(e0.elapsed_time(e1) * 1e3)
                res[name] = float(np.median(ts))
            alg = 12.0 * nnz + 4.0 * (n + 1) + 16.0 * n * k
            same = bool(torch.equal(y1[:, :k], y2[:, :k]))
            print(json.dumps(dict(k=k, tile=p["tile"], plain_us=round(res["plain"], 1), win_us=round(res["win"], 1),
                                  plain_gbs=round(alg / res["plain"] / 1e3, 1), win_gbs=round(alg / res["win"] / 1e3, 1),
                                  bit_identical=same)), flush=True)


if __name__ == "__main__":
    main()
