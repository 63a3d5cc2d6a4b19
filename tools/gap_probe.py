"""Where the device idles inside a solve: kernel timeline of one warm config-2 solve
(torch.profiler / CUPTI), idle gaps between consecutive kernels aggregated by the
kernel that follows the gap.  One JSON line + a table on stderr.

    python tools/gap_probe.py [--config 2]
"""
import argparse
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2409_05572_b200 import load  # noqa: E402
from paper_2409_05572_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="2")
args = ap.parse_args()
L = load()
w = W.config2("fix", n_ex=96) if args.config == "2" else W.config1()
a = L.from_csr(w.n, w.row_ptr, w.col, w.val)


def solve():
    return L.solve(a, w.solver, strategy=L.strategy_config(w.strategy), x0=w.x0,
                   ext=L.solve_ext(**w.ext) if w.ext else None, **w.cfg)


solve()
solve()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    r = solve()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range is not None]
ev.sort(key=lambda e: e.time_range.start)


def short(n):
    for t in ("void ", "bk::", "(anonymous namespace)::", "<unnamed>::"):
        n = n.replace(t, "")
    return n.split("<")[0].split("(")[0][:36]


busy = sum(e.time_range.end - e.time_range.start for e in ev)
span = ev[-1].time_range.end - ev[0].time_range.start
gaps = collections.defaultdict(lambda: [0, 0.0, 0.0])
for p, q in zip(ev, ev[1:]):
    g = q.time_range.start - p.time_range.end
    if g <= 0:
        continue
    k = short(p.name) + " -> " + short(q.name)
    gaps[k][0] += 1
    gaps[k][1] += g
    gaps[k][2] = max(gaps[k][2], g)
top = sorted(gaps.items(), key=lambda kv: -kv[1][1])[:25]
for k, (c, t, m) in top:
    print(f"{k:76s} {c:6d} {t / 1e3:9.2f} ms  avg {t / c:7.1f} us  max {m:8.1f} us", file=sys.stderr)
print(json.dumps({"iterations": r.iterations, "kernels": len(ev), "span_ms": span / 1e3, "busy_ms": busy / 1e3,
                  "idle_ms": (span - busy) / 1e3,
                  "big_gaps_over_20us": sum(1 for p, q in zip(ev, ev[1:]) if q.time_range.start - p.time_range.end > 20)}))
