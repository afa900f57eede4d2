"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum[,dram bytes] --csv).

  python tools/launch_summary.py launches.csv [--half]   (--half: last half of the launches only)
"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    rows = list(csv.reader(open(path)))
    hdr, data = None, collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        data.setdefault((d["ID"], d["Kernel Name"][:60]), {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    items = list(data.items())
    if "--half" in sys.argv:
        items = items[len(items) // 2:]
    agg = collections.OrderedDict()
    for (_, name), m in items:
        a = agg.setdefault(name, [0, 0.0, 0.0])
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    print(f"{'kernel':60s} {'n':>4s} {'ms':>8s} {'share':>6s} {'MB':>9s}")
    for name, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{name:60s} {a[0]:4d} {a[1] / 1e6:8.3f} {100 * a[1] / tot:5.1f}% {a[2] / 1e6:9.1f}")
    print(f"total {tot / 1e6:.3f} ms")


if __name__ == "__main__":
    main()
