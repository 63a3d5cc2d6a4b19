"""K1 SpMM probe on a BASELINE configuration's matrix: time Y = A X for a few
widths k (CUDA events, L2 flushed between calls) and print algorithmic GB/s.
Test/measurement tool only.

    python tools/spmm_probe.py --config 4 --k 160 96
"""
import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2409_05572_b200 import load, workloads as W  # noqa: E402


def matrix(cfg):
    if cfg == "2":
        return W.config2(x0=False)
    if cfg == "3":
        return W.config3(x0=False)
    if cfg == "4":
        return W.config4(x0=False)
    if cfg == "5":
        return W.config5(x0=False)
    return W.config1(x0=False)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="4")
    ap.add_argument("--k", type=int, nargs="+", default=[160])
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    w = matrix(args.config)
    full = W.full_from_lower(w.n, w.row_ptr, w.col, w.val)
    cplx = np.iscomplexobj(full.data)
    lib = load().lib
    fn = lib.bk_spmm_z if cplx else lib.bk_spmm_d
    fn.argtypes = [C.c_int] + [C.c_void_p] * 4 + [C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_void_p]
    dev = "cuda"
    rp = torch.as_tensor(full.indptr.astype(np.int32), device=dev)
    ci = torch.as_tensor(full.indices.astype(np.int32), device=dev)
    vv = torch.as_tensor(full.data.view(np.float64) if cplx else full.data, device=dev)
    nnz = full.nnz
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    out = {"workload": w.name, "n": w.n, "nnz_full": nnz, "complex": bool(cplx),
           "env": {k: v for k, v in os.environ.items() if k.startswith("BK_")}}
    es = 16 if cplx else 8
    for k in args.k:
        ld = (k + 7) // 8 * 8
        x = torch.randn(w.n, ld * (2 if cplx else 1), dtype=torch.float64, device=dev)
        y = torch.zeros_like(x)
        st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        call = lambda: fn(w.n, rp.data_ptr(), ci.data_ptr(), vv.data_ptr(), x.data_ptr(), ld, k,
                          y.data_ptr(), ld, st)
        for _ in range(2):
            assert call() == 0
        ts = []
        for _ in range(args.reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            call()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = float(np.median(ts))
        bytes_ = nnz * (es + 4) + (w.n + 1) * 4 + 2 * w.n * k * es
        gathers = nnz * k * es
        out[f"k{k}"] = {"ms": ms, "GBs": bytes_ / ms / 1e6, "gather_TBs": gathers / ms / 1e9,
                        "alg_bytes": bytes_}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
