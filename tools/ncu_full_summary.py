"""Summarise an `ncu --set full --page raw --csv` capture per kernel class.

    python tools/ncu_full_summary.py capture.csv out.json [label]

Per launch: duration, DRAM bytes read + written, SM / tensor-pipe utilisation.
Per class (the library's kernel classes: a bk_gram_d call is gram_kernel +
gram_reduce, so class traffic is the class's total DRAM bytes divided by the
number of its main-kernel launches): DRAM bytes per call — the `traffic` field
of bench.py's roofline object.
"""
import csv
import json
import sys

# main kernels of each class, real and complex (3M) forms
MAIN = {"gram": ["gram_kernel", "zgram3m_kernel"], "gemm": ["gemm_kernel", "zgemm3m_kernel"],
        "spmm": ["spmm_d_kernel", "spmm_d_half_kernel", "spmm_d_win_kernel", "spmm_z_kernel"]}
AUX = {"gram": ["gram_reduce", "zgram_reduce"]}


def short(name):
    for tok in ("(anonymous namespace)", "<unnamed>", "unnamed>", "void "):
        name = name.replace(tok, "")
    return name.split("(")[0].split("<")[0].split("::")[-1].strip()


def num(s):
    try:
        return float(s.replace(",", ""))
    except (ValueError, AttributeError):
        return None


def main():
    src, out = sys.argv[1], sys.argv[2]
    label = sys.argv[3] if len(sys.argv) > 3 else ""
    rows = list(csv.reader(open(src)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, units = rows[hi], rows[hi + 1]
    col = {h: i for i, h in enumerate(hdr)}

    def get(r, name):
        i = col.get(name)
        return num(r[i]) if i is not None and i < len(r) else None

    launches = []
    for r in rows[hi + 2:]:
        if len(r) != len(hdr):
            continue
        dur = get(r, "gpu__time_duration.sum")
        u = units[col["gpu__time_duration.sum"]] if "gpu__time_duration.sum" in col else "ns"
        if dur is not None and u in ("ns", "nsecond"):
            dur /= 1e3
        elif dur is not None and u in ("ms", "msecond"):
            dur *= 1e3
        rd = get(r, "dram__bytes_read.sum") or 0.0
        wr = get(r, "dram__bytes_write.sum") or 0.0
        for name, scale in (("dram__bytes_read.sum", rd), ("dram__bytes_write.sum", wr)):
            un = units[col[name]] if name in col else "byte"
            f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(un, 1)
            if name.endswith("read.sum"):
                rd = scale * f
            else:
                wr = scale * f
        launches.append({"kernel": short(r[col["Kernel Name"]]), "us": dur, "dram_bytes": rd + wr,
                         "sm_pct": get(r, "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
                         "dram_pct": get(r, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")})
    classes = {}
    for cls, main_k in MAIN.items():
        # the library's K2/K3 classes count only the n-row contractions; the
        # eigensolver's and the HL trick's coefficient-space ones (d rows) move
        # < 4 MB and are excluded here too (their reduce launches follow them)
        mains, members = [], []
        for idx, x in enumerate(launches):
            if x["kernel"] not in main_k or x["dram_bytes"] < 4e6:
                continue
            mains.append(x)
            members.append(x)
            nxt = launches[idx + 1] if idx + 1 < len(launches) else None
            if nxt and nxt["kernel"] in AUX.get(cls, []):
                members.append(nxt)
        if not mains:
            continue
        classes[cls] = {
            "calls": len(mains),
            "dram_bytes_per_launch": sum(x["dram_bytes"] for x in members) / len(mains),
            "us_per_call": sum(x["us"] or 0 for x in members) / len(mains),
            "main_kernel_sm_pct_mean": sum(x["sm_pct"] or 0 for x in mains) / len(mains),
        }
    json.dump({"source": src, "label": label, "launches": launches, "classes": classes}, open(out, "w"), indent=1)
    print(json.dumps(classes, indent=1))


if __name__ == "__main__":
    main()
