#!/usr/bin/env python
"""Per-degree ms table of A/B bench runs: python tools/ab_table.py gpurun_out/TAG_*.jsonl"""
import json, sys, collections
for f in sys.argv[1:]:
    per = collections.defaultdict(list)
    for line in open(f):
        line = line.strip()
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        for e in d.get("per_degree", []):
            per[e["p"]].append((e["ms"], e["roofline_frac"]))
    cells = []
    for p in sorted(per):
        ms = sorted(x[0] for x in per[p])
        fr = max(x[1] for x in per[p])
        cells.append("p%d %.4f (%.2f)" % (p, ms[len(ms) // 2], fr))
    print("%-40s %s" % (f.split("/")[-1], "  ".join(cells)))
