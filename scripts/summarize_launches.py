"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel share."""
import collections
import csv
import sys

UNIT = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    mi = h.index("Metric Name")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)
        name = r[ki].split("(")[0].replace("kgq::<unnamed>::", "kgq::")[:70]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"# {path}: {sum(v[0] for v in agg.values())} launches, {tot:.1f} us total "
          "(ncu serialised, cold-cache: compare shares, not absolutes)")
    print(f"{'us':>12} {'share':>6} {'n':>5}  kernel")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{v[1]:12.1f} {100 * v[1] / tot:5.1f}% {v[0]:5d}  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
