"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv) of tools/prof_build.py: per-kernel time and DRAM bytes, one build
(the first of the process's builds is dropped when two are present)."""
import collections
import csv
import sys

TU = {"msecond": 1.0, "ms": 1.0, "usecond": 1e-3, "us": 1e-3, "nsecond": 1e-6, "ns": 1e-6}
BU = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, rows = rows[0], rows[1:]
    ki, mi, vi, ui = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    agg = collections.defaultdict(lambda: [set(), 0.0, 0.0])
    for r in rows:
        k = r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", "").replace("sl::", "")
        v = float(r[vi].replace(",", ""))
        a = agg[k]
        a[0].add(r[hdr.index("ID")])
        if r[mi] == "gpu__time_duration.sum":
            a[1] += v * TU[r[ui]]
        else:
            a[2] += v * BU[r[ui]]
    tot_t = sum(a[1] for a in agg.values())
    tot_b = sum(a[2] for a in agg.values())
    print(f"| kernel | launches | ms | DRAM GB |\n|---|---|---|---|")
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| {k} | {len(a[0])} | {a[1]:.4f} | {a[2] / 1e9:.3f} |")
    print(f"| total | | {tot_t:.4f} | {tot_b / 1e9:.3f} |")


if __name__ == "__main__":
    main(sys.argv[1])
