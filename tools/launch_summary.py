"""Summarise an ncu --csv launch list (gpu__time_duration.sum): per kernel
name, launches, total and average time, share.  usage: launch_summary.py FILE"""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = []
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "nsecond")
        scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}.get(unit, 1e-3)
        name = r["Kernel Name"][:60]
        tot[name] += v * scale
        cnt[name] += 1
    all_us = sum(tot.values())
    print(f"{'kernel':60s} {'launches':>8s} {'total ms':>10s} {'avg us':>9s} share")
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"{k:60s} {cnt[k]:8d} {tot[k] / 1e3:10.3f} {tot[k] / cnt[k]:9.2f} {tot[k] / all_us:.3f}")
    print(f"total {all_us / 1e3:.3f} ms over {sum(cnt.values())} launches")


if __name__ == "__main__":
    main(sys.argv[1])
