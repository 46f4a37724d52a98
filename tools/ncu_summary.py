"""Summaries of ncu evidence under profiles/ (diagnostics, not product code).

    python tools/ncu_summary.py traffic <raw.csv> <key> [<key> ...]   # -> profiles/ncu_traffic.json
    python tools/ncu_summary.py launches <launches.csv>               # per-kernel launch table

`traffic`: reads an `ncu --set full` capture exported with `ncu -i X --page raw --csv` and
stores dram__bytes_read.sum + dram__bytes_write.sum of its (single) launch under each key of
profiles/ncu_traffic.json, with the kernel name and source file (bench.py's roofline.traffic).
`launches`: the `--metrics gpu__time_duration.sum` launch list: count, mean and share of the
total device time per kernel.
"""
import csv
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def traffic(path, keys):
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    get = lambda m: float(vals[hdr.index(m)]) * UNIT[units[hdr.index(m)]]  # noqa: E731
    total = get("dram__bytes_read.sum") + get("dram__bytes_write.sum")
    out_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    d = json.load(open(out_path)) if os.path.exists(out_path) else {}
    for k in keys:
        d[k] = int(round(total))
        d[f"_{k}"] = {"kernel": vals[hdr.index("Kernel Name")], "source": os.path.relpath(path, ROOT),
                      "dram_read": get("dram__bytes_read.sum"),
                      "dram_write": get("dram__bytes_write.sum"),
                      "duration_us": float(vals[hdr.index("gpu__time_duration.sum")])}
    d["_about"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant kernel "
                   "from one `ncu --set full` capture (cold L2 per replay: lines still dirty in L2 at "
                   "the kernel's end are not written back inside the launch); see the `_<key>` "
                   "entries for the kernel and the capture file")
    json.dump(d, open(out_path, "w"), indent=1)
    print(json.dumps(d, indent=1))


def launches(path):
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    t = defaultdict(list)
    for r in rows[1:]:
        if r[mi] == "gpu__time_duration.sum":
            t[r[ki]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in t.values())
    for k, v in sorted(t.items(), key=lambda kv: -sum(kv[1])):
        print(f"{len(v):5d} x {sum(v) / len(v) / 1e3:9.2f} us  share {sum(v) / tot:6.1%}  {k[:100]}")


if __name__ == "__main__":
    if sys.argv[1] == "traffic":
        traffic(sys.argv[2], sys.argv[3:])
    else:
        launches(sys.argv[2])
