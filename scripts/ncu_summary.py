"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel launch counts, total and mean device time, share of the total."""
import csv
import re
import sys
from collections import defaultdict


def short(name):
    name = re.sub(r"\(.*", "", name)
    name = re.sub(r"^void ", "", name)
    name = re.sub(r"svtb::(_GLOBAL__N__\w+::)?", "", name)
    return name[:60]


def main(path, top=25):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rdr = csv.DictReader(lines)
    for r in rdr:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}.get(unit, 1e-3)
        rows.append((short(r["Kernel Name"]), v * scale))
    agg = defaultdict(lambda: [0, 0.0])
    for k, us in rows:
        agg[k][0] += 1
        agg[k][1] += us
    tot = sum(v[1] for v in agg.values())
    print(f"{len(rows)} launches, {tot/1e3:.2f} ms device time")
    print(f"{'kernel':60s} {'launches':>8s} {'total_ms':>10s} {'mean_us':>9s} {'share':>6s}")
    for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{k:60s} {n:8d} {us/1e3:10.3f} {us/n:9.2f} {100*us/tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
