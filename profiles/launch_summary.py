"""Per-kernel totals of an `ncu --metrics gpu__time_duration.sum --csv` launch list.

    python profiles/launch_summary.py launches.csv

Cold-cache, serialised launches (ncu replays each kernel alone): compare each kernel's SHARE of
the step with the live CUDA-event timing, not the absolute times.
"""
import collections
import csv
import sys


def main(path):
    rows = [r for r in csv.DictReader(l for l in open(path) if not l.startswith("=="))
            if r.get("Metric Name") == "gpu__time_duration.sum"]
    agg = collections.OrderedDict()
    for r in rows:
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        us = v / 1000.0 if unit in ("nsecond", "ns") else (v * 1000.0 if unit in ("msecond", "ms") else v)
        name = r["Kernel Name"].split("(")[0][:44]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += us
    tot = sum(a[1] for a in agg.values()) or 1.0
    print(f"source: {path} (cold-cache, serialised launches: compare shares, not absolute times)")
    for name, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name:46s} n={n:4d} total={us:10.1f} us  mean={us / n:9.1f} us  share={100 * us / tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
