"""Summarise A/B bench logs: python scripts/ab_table.py gpurun_out/ab_*.log"""
import json
import sys
from collections import defaultdict

rows = defaultdict(list)
for f in sys.argv[1:]:
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line)
            key = f.rsplit("/", 1)[-1].rsplit("_", 1)[0]
            rows[key].append((d["ms_per_step"], d["roofline"]["k1_ms"]))
for k in sorted(rows):
    v = rows[k]
    print(f"{k:28s} step " + " ".join(f"{a:7.2f}" for a, _ in v) + "   k1 " + " ".join(f"{b:7.2f}" for _, b in v))
