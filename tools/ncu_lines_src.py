"""Per-source-line hot spots of one kernel in a --import-source ncu report.
  python tools/ncu_lines_src.py gpurun_out/x.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, fname, hdr = [], None, None
for r in csv.reader(io.StringIO(raw)):
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit() or len(r) < len(hdr):
        continue
    try:  # per-line aggregate rows have Address "-"
        samp = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        inst = int(r[hdr.index("Instructions Executed")] or 0)
    except ValueError:
        continue
    if samp or inst:
        rows.append((samp, inst, fname, int(r[0]), r[1].strip()[:90]))
ts = sum(r[0] for r in rows) or 1
ti = sum(r[1] for r in rows) or 1
print(f"total samples {ts}  total warp-instr {ti:.3e}")
for s, i, f, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{100*s/ts:5.1f}% smp {100*i/ti:5.1f}% ins  {f}:{ln:<5} {src}")
