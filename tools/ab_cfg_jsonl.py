#!/usr/bin/env python
"""Side-by-side ms / roofline frac of bench_configs.py JSONL files:
    python tools/ab_cfg_jsonl.py A.jsonl B.jsonl ..."""
import json
import sys

rows = {}
for f in sys.argv[1:]:
    for line in open(f):
        line = line.strip()
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        rows.setdefault((d.get("config"), d.get("p")), {})[f] = (d.get("ms"), d.get("roofline_frac"))
print("%-8s %3s " % ("config", "p") + " ".join("%22s" % f.split("/")[-1][-22:] for f in sys.argv[1:]))
for k in sorted(rows, key=lambda k: (str(k[0]), k[1] or 0)):
    print("%-8s %3s " % k + " ".join("%12s %9s" % rows[k].get(f, ("-", "-")) for f in sys.argv[1:]))
