"""Summarise tools/ab.sh output: one line per (lib, case) with qps for each sweep entry."""
import json
import re
import sys

for line in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/t.log"):
    m = re.match(r"^(\S+ c\d+ k\d+) (.*)$", line.strip())
    if not m:
        print(line.rstrip())
        continue
    objs = re.findall(r'\{"env".*?"qps": [0-9.e+]+\}', m.group(2))
    parts = []
    for o in objs:
        d = json.loads(o)
        parts.append(f"{d['env'] or 'default'}: {d['qps']:.0f} (kernel {d['kernel_ms']:.2f} ms)")
    print(m.group(1), " | ".join(parts))
