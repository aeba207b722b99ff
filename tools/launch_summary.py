"""Per-kernel totals of `ncu --metrics gpu__time_duration.sum --csv` launch
lists: python tools/launch_summary.py launches.csv [more.csv ...]"""
import collections
import csv
import sys

for f in sys.argv[1:]:
    try:
        rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    except OSError:
        continue
    h = rows[0]
    ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    data = [(r[ki], float(r[vi])) for r in rows[1:] if r[mi] == "gpu__time_duration.sum"]
    c = collections.defaultdict(lambda: [0, 0.0])
    for k, v in data:
        c[k][0] += 1
        c[k][1] += v
    tot = sum(v for _, v in data) or 1.0
    print(f"== {f}: {len(data)} launches, {tot / 1e6:.3f} ms total (ncu, cold-cache, serialised)")
    print(f"{'kernel':64s} {'launches':>8s} {'ms':>10s} {'share':>6s} {'us/launch':>10s}")
    for k, (n, v) in sorted(c.items(), key=lambda x: -x[1][1]):
        print(f"{k[:64]:64s} {n:8d} {v / 1e6:10.3f} {100 * v / tot:5.1f}% {v / n / 1e3:10.1f}")
    print()
