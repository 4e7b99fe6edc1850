#!/usr/bin/env python
"""Per-degree median ms of bench_configs A/B runs:
python tools/ab_cfg_table.py gpurun_out/TAG_*.jsonl"""
import collections, json, sys
for f in sys.argv[1:]:
    per = collections.defaultdict(list)
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line)
            per[(d.get("config"), d.get("p"))].append(d["ms"])
    cells = ["%s p%d %.4f" % (c, p, sorted(v)[len(v) // 2]) for (c, p), v in sorted(per.items())]
    print("%-28s %s" % (f.split("/")[-1], "  ".join(cells)))
