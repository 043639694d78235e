"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per kernel name, launches and total us (ncu times: cold, serialised).
    python tools/launch_summary.py launches.csv [top]"""
import collections
import csv
import sys


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if r[ki] == "Kernel Name":
            continue
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        agg[r[ki].split("(")[0][:70]][0] += 1
        agg[r[ki].split("(")[0][:70]][1] += v
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{c:4d} {t:9.1f} us  {n}")
    print("launches", sum(c for c, _ in agg.values()), "sum_us", round(sum(t for _, t in agg.values()), 1))


if __name__ == "__main__":
    main()
