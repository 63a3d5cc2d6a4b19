"""Measure FP64 peaks on the GPU box (cuBLAS DGEMM/ZGEMM via torch) and host info.

Writes gpurun_out/fp64_peaks.json. Run under gpurun; not part of the product path.
"""
import json, os, subprocess, time
import torch

def bench(fn, iters=10):
    best = 1e9
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    for _ in range(iters):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    return best

out = {}
props = torch.cuda.get_device_properties(0)
out["gpu"] = props.name
out["sm_count"] = props.multi_processor_count
out["l2_bytes"] = getattr(props, "L2_cache_size", None)
N = 8192
a = torch.randn(N, N, dtype=torch.float64, device="cuda")
b = torch.randn(N, N, dtype=torch.float64, device="cuda")
t = bench(lambda: torch.matmul(a, b))
out["dgemm_tflops_burst"] = 2 * N**3 / t / 1e12
# sustained 4 s
torch.cuda.synchronize(); t0 = time.time(); cnt = 0
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
s.record()
while time.time() - t0 < 4.0:
    torch.matmul(a, b); cnt += 1
    if cnt % 4 == 0: torch.cuda.synchronize()
e.record(); torch.cuda.synchronize()
out["dgemm_tflops_sustained"] = 2 * N**3 * cnt / (s.elapsed_time(e) / 1e3) / 1e12
del a, b
M = 4096
za = torch.randn(M, M, dtype=torch.complex128, device="cuda")
zb = torch.randn(M, M, dtype=torch.complex128, device="cuda")
t = bench(lambda: torch.matmul(za, zb))
out["zgemm_tflops_burst"] = 8 * M**3 / t / 1e12
del za, zb
# tall-skinny Gram via cuBLAS (n=262144, d=288): reference point for K2
n, d = 262144, 288
x = torch.randn(n, d, dtype=torch.float64, device="cuda")
t = bench(lambda: x.t() @ x)
out["cublas_gram_262144x288_tflops"] = 2 * n * d * d / t / 1e12
c = torch.randn(d, 96, dtype=torch.float64, device="cuda")
t = bench(lambda: x @ c)
out["cublas_update_262144x288x96_tflops"] = 2 * n * d * 96 / t / 1e12
# HBM copy fp64
big = torch.empty(2**28, dtype=torch.float64, device="cuda"); big2 = torch.empty_like(big)
t = bench(lambda: big2.copy_(big))
out["copy_gbs"] = 2 * big.numel() * 8 / t / 1e9
out["host_nproc"] = os.cpu_count()
try:
    out["host_cpu"] = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
except Exception:
    pass
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/fp64_peaks.json", "w"), indent=1)
print(json.dumps(out, indent=1))
