"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
launches and average duration per kernel, sorted by total time.

    python tools/launch_summary.py launches.csv [TITLE] > summary.txt
"""
import collections
import csv
import sys


def main():
    rows = list(csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")))
    h = rows[0]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    ui = h.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in rows[1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            v = float(r[vi].replace(",", ""))
            v *= {"ns": 1e-3, "us": 1.0, "ms": 1e3, "usecond": 1.0, "nsecond": 1e-3, "msecond": 1e3}.get(r[ui], 1.0)
            agg[r[ki]].append(v)
    if len(sys.argv) > 2:
        print(sys.argv[2])
        print()
    tot = sum(sum(v) for v in agg.values())
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k[:76]:76s} launches {len(v):3d}  avg {sum(v) / len(v):10.1f} us  share {100 * sum(v) / tot:5.1f}%")


if __name__ == "__main__":
    main()
