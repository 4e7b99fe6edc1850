#!/usr/bin/env python
"""Executed warp-instruction mix by SASS opcode from an ncu report:
    python tools/ncu_opmix.py REPORT [top]"""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Address")
iS, iE, iW = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
ops, stall = collections.Counter(), collections.Counter()
for r in rows:
    if len(r) != len(hdr) or r[0] == "Address":
        continue
    toks = r[iS].split()
    if toks and toks[0].startswith("@"):
        toks = toks[1:]
    if not toks:
        continue
    op = toks[0].split(".")[0]
    if op in ("LDS", "STS", "LDG", "STG"):
        op = ".".join(toks[0].split(".")[:1] + [t for t in toks[0].split(".")[1:] if t in ("64", "128")])
    ops[op] += int(r[iE])
    stall[op] += int(r[iW])
tot, st = sum(ops.values()), sum(stall.values()) or 1
print("total warp instructions %d" % tot)
for op, c in ops.most_common(top):
    print("%-10s %12d %5.1f%%   stall samples %5.1f%%" % (op, c, 100.0 * c / tot, 100.0 * stall[op] / st))
