"""profiles/traffic.json from an ncu launch list with DRAM metrics:

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \\
        --clock-control none --csv --log-file traffic_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu --pyc 0
    python tools/traffic_json.py c3 traffic_c3.csv [more workload/csv pairs]

Per kernel: mean (read + write) bytes per launch over the captured launches.
"""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def parse(path):
    per = collections.defaultdict(lambda: collections.defaultdict(float))
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        name = r["Kernel Name"].split("(")[0]
        if not name.startswith("upy_"):
            continue
        key = (r["ID"], name)
        unit = r.get("Metric Unit", "")
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
                 "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)
        per[key][r["Metric Name"]] += v * scale
    out = collections.defaultdict(list)
    for (_, name), m in per.items():
        out[name].append(m)
    res = {}
    for name, ms in out.items():
        b = [m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"] for m in ms]
        t = [m["gpu__time_duration.sum"] for m in ms]
        res[name] = {"bytes_per_launch": sum(b) / len(b), "seconds_per_launch": sum(t) / len(t), "launches": len(b)}
    return res


def main(argv):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    d = json.load(open(p)) if os.path.exists(p) else {}
    for wl, path in zip(argv[0::2], argv[1::2]):
        d[wl] = parse(path)
    with open(p, "w") as f:
        json.dump(d, f, indent=1)
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    main(sys.argv[1:])
