"""Summarise an ncu source page (--page source --csv --print-source=cuda,sass) per CUDA line:
stall samples and instructions executed. Usage: python tools/ncu_lines.py src.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
fname, out, tot_s, tot_i = "", [], 0, 0
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0] not in ("", "Line No", "Function Name") and r[2] == "-":
        try:
            s, i = int(r[4]), int(r[7])
        except ValueError:
            continue
        out.append((s, i, f"{fname}:{r[0]}", r[1][:90]))
        tot_s += s
        tot_i += i
for s, i, loc, src in sorted(out, reverse=True)[:top]:
    print(f"{100*s/max(tot_s,1):5.1f}% samp {100*i/max(tot_i,1):5.1f}% inst  {loc:22s} {src}")
