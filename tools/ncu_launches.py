"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list by kernel."""
import collections
import csv
import sys

UNIT = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
        "s": 1e3, "second": 1e3}


def summarize(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * UNIT[r[ui]]
    tot = sum(a[1] for a in agg.values())
    lines = [f"{'kernel':44s} {'launches':>8s} {'total ms':>10s} {'share':>7s}"]
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{k:44s} {c:8d} {t:10.3f} {100 * t / tot:6.2f}%")
    lines.append(f"{'TOTAL':44s} {sum(a[0] for a in agg.values()):8d} {tot:10.3f}")
    return "\n".join(lines)


if __name__ == "__main__":
    print(summarize(sys.argv[1]))
