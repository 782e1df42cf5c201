"""Summarise bench.py's per-layer list by layer role (tools; reads a bench log)."""
import json
import signal
import re
import sys
from collections import defaultdict

signal.signal(signal.SIGPIPE, signal.SIG_DFL)

d = None
for line in open(sys.argv[1]):
    if line.startswith("{"):
        d = json.loads(line)
print("value", d["value"], d["unit"], "ms/step", d["ms_per_step"])
agg = defaultdict(lambda: [0, 0.0, 0.0])
for x in d.get("layers", []):
    k = re.sub(r"s\db\d+_", "", x["name"]) if x["kind"] == "conv" else x["kind"] + ":" + re.sub(r"\d", "", x["name"])
    agg[k][0] += 1
    agg[k][1] += x["ms"]
    agg[k][2] += x["ms"] * x.get("gflops", 0)
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda t: -t[1][1]):
    print(f"{k:20s} n={v[0]:3d} ms={v[1]:7.2f} ({v[1] / tot * 100:4.1f}%) TF={v[2] / max(v[1], 1e-9) / 1e3:6.1f}")
if len(sys.argv) > 2:
    for x in d.get("layers", []):
        print(x["name"], x["ms"], round(x.get("gflops", 0) / 1e3, 1))
