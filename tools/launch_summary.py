"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into a markdown table.

usage: python tools/launch_summary.py gpurun_out/r1_launches.csv [title] > profiles/r01_launches.md
"""
import csv
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else path
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[start]
    agg = defaultdict(lambda: [0, 0.0])
    order = []
    for r in rows[start + 1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0].replace("(anonymous namespace)::", "").replace("unnamed>::", "")
        unit = d.get("Metric Unit", "ns")
        v = float(d["Metric Value"].replace(",", ""))
        v *= {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1e-3)
        agg[k][0] += 1
        agg[k][1] += v
        order.append((k, v))
    tot = sum(v[1] for v in agg.values())
    print(f"# Launch list: {title}\n")
    print(f"{len(order)} launches, {tot / 1e3:.2f} ms of serialised kernel time "
          "(ncu, --clock-control none, cold caches: shares matter, not absolutes).\n")
    print("| kernel | launches | total ms | share | mean us |")
    print("|---|---:|---:|---:|---:|")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{k}` | {n} | {t / 1e3:.3f} | {100 * t / tot:.1f}% | {t / n:.1f} |")


if __name__ == "__main__":
    main()
