"""Summarise ncu output for profiles/: a --set full report (.ncu-rep) and/or a launch list
(--metrics gpu__time_duration.sum --csv). Writes JSON + a short markdown table.

  python tools/ncu_summary.py --rep gpurun_out/x.ncu-rep --launches gpurun_out/l.csv --out profiles/r01_c2
"""
import argparse
import csv
import io
import json
import subprocess
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "l1tex__t_bytes.sum", "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]


def rep_summary(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    out = []
    for v in rows[2:]:
        d = {"kernel": v[h.index("Kernel Name")][:120]}
        for k in KEYS:
            if k in h:
                i = h.index(k)
                d[k] = f"{v[i]} {units[i]}".strip()
        stalls = {}
        for i, k in enumerate(h):
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    stalls[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(v[i].replace(",", ""))
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1.0
        d["stall_pct"] = {k: round(100 * x / tot, 1) for k, x in sorted(stalls.items(), key=lambda x: -x[1])[:8]}
        out.append(d)
    return out


def launches_summary(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("sl::<unnamed>::", "")
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6)
    tot = sum(v[1] for v in agg.values())
    return [{"kernel": n, "launches": c, "ms": round(ms, 4), "share_pct": round(100 * ms / tot, 2)}
            for n, (c, ms) in sorted(agg.items(), key=lambda x: -x[1][1])]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--out", required=True)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    res = {"note": a.note}
    md = [f"# {a.out.split('/')[-1]}", "", a.note, ""]
    if a.rep:
        res["full"] = rep_summary(a.rep)
        for d in res["full"]:
            md += [f"## {d['kernel']}", "", "| metric | value |", "|---|---|"]
            md += [f"| {k} | {v} |" for k, v in d.items() if k not in ("kernel", "stall_pct")]
            md += ["", "stall reasons (% of samples): " + ", ".join(f"{k} {v}" for k, v in d["stall_pct"].items()), ""]
    if a.launches:
        res["launches"] = launches_summary(a.launches)
        md += ["## launch list (ncu, cold-cache serialised: compare shares)", "", "| kernel | launches | ms | share |",
               "|---|---|---|---|"]
        md += [f"| {d['kernel']} | {d['launches']} | {d['ms']} | {d['share_pct']}% |" for d in res["launches"]]
    json.dump(res, open(a.out + ".json", "w"), indent=1)
    open(a.out + ".md", "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
