"""Summarise an ncu --csv launch list (gpu__time_duration.sum): one line per
kernel name with count, mean and total microseconds.

    python scripts/ncu_times.py launches.csv
"""
import collections
import csv
import sys


def main():
    rows = [r for r in csv.DictReader(l for l in open(sys.argv[1]) if l.startswith('"'))]
    agg = collections.OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        agg.setdefault(r["Kernel Name"][:80], []).append(float(r["Metric Value"]) / 1e3)
    for k, v in agg.items():
        print(f"{len(v):4d} x {sum(v) / len(v):10.1f} us  (total {sum(v):10.1f})  {k}")


if __name__ == "__main__":
    main()
