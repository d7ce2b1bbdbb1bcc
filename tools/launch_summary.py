"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV):
per-kernel launch count, mean and total duration, share of the total."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    d = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi and r[vi]:
            d[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0))
    tot = sum(sum(v) for v in d.values())
    print(f"{path}: {sum(len(v) for v in d.values())} launches, {tot:.1f} us total (cold-cache, serialised)")
    print(f"{'kernel':58s} {'n':>5s} {'mean us':>9s} {'total us':>10s} {'share':>6s}")
    for k, v in sorted(d.items(), key=lambda t: -sum(t[1])):
        print(f"{k[:58]:58s} {len(v):5d} {sum(v)/len(v):9.2f} {sum(v):10.1f} {100*sum(v)/tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
