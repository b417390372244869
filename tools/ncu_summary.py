"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list per kernel (dev tool).

usage: python tools/ncu_summary.py launches.csv [source-note] > summary.json
"""
import csv
import json
import re
import sys
from collections import defaultdict

UNIT = {"ns": 1e-3, "nsecond": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}


def short(name: str) -> str:
    m = re.search(r"(k_[A-Za-z0-9_]+)", name)
    return m.group(1) if m else name.split("(")[0]


def main() -> None:
    path = sys.argv[1]
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(lines[start:]))
    acc = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        us = float(r["Metric Value"].replace(",", "")) * UNIT.get(r["Metric Unit"], 1.0)
        a = acc[short(r["Kernel Name"])]
        a[0] += 1
        a[1] += us
    total = sum(v[1] for v in acc.values())
    out = {
        "source": sys.argv[2] if len(sys.argv) > 2 else path,
        "total_us": round(total, 1),
        "kernels": {
            k: {"launches": n, "total_us": round(t, 1), "mean_us": round(t / n, 1), "share": round(t / total, 4)}
            for k, (n, t) in sorted(acc.items(), key=lambda kv: -kv[1][1])
        },
    }
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
