"""Convert an `ncu --metrics ... --csv --log-file` capture (one row per launch and
metric) into the per-launch / per-class JSON that bench.py reads for `traffic`
(same schema as tools/ncu_full_summary.py's output).

    python tools/ncu_long_to_json.py capture.csv out.json [label]
"""
import collections
import csv
import json
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from ncu_full_summary import AUX, MAIN, short  # noqa: E402

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3, "us": 1.0,
        "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def main():
    src, out = sys.argv[1], sys.argv[2]
    label = sys.argv[3] if len(sys.argv) > 3 else ""
    rows = [r for r in csv.reader(open(src)) if len(r) == 15 and r[0] != "ID"]
    per = collections.OrderedDict()
    for r in rows:
        d = per.setdefault(int(r[0]), {"kernel": short(r[4]), "us": None, "dram_bytes": 0.0,
                                       "sm_pct": None, "dram_pct": None})
        v = float(r[14].replace(",", "")) * UNIT.get(r[13], 1.0)
        if r[12] == "gpu__time_duration.sum":
            d["us"] = v
        elif r[12].startswith("dram__bytes_"):
            d["dram_bytes"] += v
    launches = list(per.values())
    classes = {}
    for cls, main_k in MAIN.items():
        mains, members = [], []
        for idx, x in enumerate(launches):
            if x["kernel"] != main_k or x["dram_bytes"] < 4e6:
                continue
            mains.append(x)
            members.append(x)
            nxt = launches[idx + 1] if idx + 1 < len(launches) else None
            if nxt and nxt["kernel"] in AUX.get(cls, []):
                members.append(nxt)
        if mains:
            classes[cls] = {"calls": len(mains), "dram_bytes_per_launch": sum(m["dram_bytes"] for m in members)
                            / len(mains), "us_per_call": sum(m["us"] or 0 for m in members) / len(mains)}
    json.dump({"source": src, "label": label, "launches": launches, "classes": classes}, open(out, "w"), indent=1)
    print(json.dumps(classes))


if __name__ == "__main__":
    main()
