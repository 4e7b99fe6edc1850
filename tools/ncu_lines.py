#!/usr/bin/env python
"""Per-source-line stall samples from an ncu report (needs -lineinfo):
    python tools/ncu_lines.py REPORT [top]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname = None
agg = {}
tot = 0
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0] not in ("", "Line No") and r[2] == "-":
        try:
            s = int(r[4])
        except ValueError:
            continue
        key = (fname, int(r[0]), r[1].strip()[:70])
        agg[key] = agg.get(key, 0) + s
        tot += s
for (f, ln, src), s in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print("%5.1f%%  %s:%d  %s" % (100.0 * s / max(tot, 1), f, ln, src))
