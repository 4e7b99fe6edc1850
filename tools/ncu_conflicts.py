#!/usr/bin/env python
"""Per-source-line shared-memory wavefronts (total / excessive) from an ncu
report: python tools/ncu_conflicts.py REPORT [top]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
hdr, f, res = None, None, []
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) > 20 and r[2] == "-":
        d = dict(zip(hdr, r))
        try:
            ex, wf = int(d["L1 Wavefronts Shared Excessive"]), int(d["L1 Wavefronts Shared"])
        except (KeyError, ValueError):
            continue
        if wf:
            res.append((ex, wf, f, r[0], r[1].strip()[:70]))
tot = sum(x[1] for x in res)
exs = sum(x[0] for x in res)
print("shared wavefronts %d, excessive %d (%.0f%%)" % (tot, exs, 100.0 * exs / max(tot, 1)))
for ex, wf, f, ln, src in sorted(res, reverse=True)[:top]:
    print("%10d / %10d  %s:%s  %s" % (ex, wf, f, ln, src))
