"""GPU idle time inside one config-2 solve, from a CUPTI trace (torch.profiler):
sums the gaps between consecutive kernels on the device and attributes each gap
to the kernel that precedes it.  Tuning tool (the profiler perturbs timing a
little; the shape of the gaps is what matters)."""
import collections
import json
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2409_05572_b200 import load, workloads as W  # noqa: E402


def short(name):
    for tok in ("(anonymous namespace)", "<unnamed>", "unnamed>", "void "):
        name = name.replace(tok, "")
    return name.split("(")[0].split("<")[0].split("::")[-1]


def main():
    L = load()
    w = W.config2("fix")
    a = L.from_csr(w.n, w.row_ptr, w.col, w.val)
    a.norm_est()
    run = lambda: L.solve(a, w.solver, strategy=L.strategy_config(w.strategy), x0=w.x0, **w.cfg)
    run()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        r = run()
        torch.cuda.synchronize()
    path = os.path.join(tempfile.gettempdir(), "trace.json")
    prof.export_chrome_trace(path)
    ev = json.load(open(path))["traceEvents"]
    k = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e],
               key=lambda e: e["ts"])
    busy = sum(e["dur"] for e in k)
    span = k[-1]["ts"] + k[-1]["dur"] - k[0]["ts"]
    gaps = collections.Counter()
    count = collections.Counter()
    for p, q in zip(k, k[1:]):
        g = q["ts"] - (p["ts"] + p["dur"])
        if g > 0:
            key = f"{short(p['name'])} -> {short(q['name'])}"
            gaps[key] += g
            count[key] += 1
    print(json.dumps({"iterations": r.iterations, "span_ms": span / 1e3, "busy_ms": busy / 1e3,
                      "idle_ms": (span - busy) / 1e3, "kernels": len(k)}))
    for key, g in gaps.most_common(15):
        print(f"{g / 1e3:9.2f} ms  {count[key]:6d}x  {key}")
    # one steady-state iteration (between two tridiagonalisations), launch by launch
    tri = [i for i, e in enumerate(k) if "tridiag" in e["name"]]
    if len(tri) > 101:
        for e in k[tri[100]:tri[101] + 1]:
            a = e.get("args", {})
            print(f"  {short(e['name'])[-24:]:24s} {str(a.get('grid')):>16s} {str(a.get('block')):>14s} {e['dur']:9.1f} us"
                  f"  {e['name'].split('(')[0][-60:] if 'kernel<' in e['name'] else ''}")
    # device time per kernel (CUPTI durations, concurrent-free stream)
    per = collections.defaultdict(lambda: [0, 0.0])
    for e in k:
        per[short(e["name"])][0] += 1
        per[short(e["name"])][1] += e["dur"]
    print(f"{'kernel':32s} {'launches':>8s} {'total_ms':>9s} {'avg_us':>8s}")
    for name, (c, d) in sorted(per.items(), key=lambda x: -x[1][1])[:30]:
        print(f"{name[-32:]:32s} {c:8d} {d / 1e3:9.2f} {d / c:8.2f}")


if __name__ == "__main__":
    main()
