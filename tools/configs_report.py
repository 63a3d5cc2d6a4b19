"""Summarise tools/run_config.py --out JSON files into a markdown table.

    python tools/configs_report.py out.md run1.json run2.json ...
"""
import json
import sys


def main():
    out, files = sys.argv[1], sys.argv[2:]
    lines = ["| workload | status | iterations | seconds | s / iteration | final r | n_now trajectory (run-length) | "
             "kernel ms (spmm / gram / gemm / syev / chol) | GB/s spmm, TF/s gram, gemm |",
             "|---|---|---|---|---|---|---|---|---|"]
    for f in files:
        try:
            d = json.load(open(f))
        except (OSError, ValueError) as e:
            lines.append(f"| {f} | unreadable: {e} | | | | | | | |")
            continue
        ks = d.get("kernel_stats") or {}
        def k(name, i):
            v = ks.get(name)
            return v[i] if v else 0.0
        ms = " / ".join(f"{k(n, 1):.0f}" for n in ("spmm", "gram", "gemm", "syev", "chol"))
        rates = []
        for n, kind in (("spmm", "b"), ("gram", "f"), ("gemm", "f")):
            t = k(n, 1)
            if t:
                rates.append(f"{(k(n, 2) / t / 1e6):.0f}" if kind == "b" else f"{(k(n, 3) / t / 1e9):.1f}")
            else:
                rates.append("-")
        rle = d.get("n_now_rle", [])
        traj = ", ".join(f"{w}x{c}" for w, c in rle[:8]) + (" ..." if len(rle) > 8 else "")
        status = {0: "converged", 1: "max_iters", 2: "stagnated"}.get(d.get("status"), str(d.get("status")))
        it = d.get("iterations") or 1
        lines.append(f"| {d.get('workload')} | {status} | {d.get('iterations')} | {d.get('seconds', 0):.1f} | "
                     f"{d.get('seconds', 0) / it * 1e3:.1f} ms | {d.get('final_r', 0):.2e} | {traj} | {ms} | "
                     f"{', '.join(rates)} |")
    with open(out, "w") as fh:
        fh.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
