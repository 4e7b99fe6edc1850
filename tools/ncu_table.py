#!/usr/bin/env python
"""One table over several ncu summaries (profiles/*.md written by
tools/ncu_summary.py): python tools/ncu_table.py OUT.md LABEL=profiles/x.md ..."""
import re
import sys

KEYS = [("duration", "duration"), ("FP64 pipe active %", "FP64 pipe %"), ("DMMA pipe %", "DMMA %"),
        ("issue active %", "issue %"), ("achieved occupancy %", "occupancy %"),
        ("registers/thread", "regs"), ("DRAM read", "DRAM read"), ("DRAM write", "DRAM write")]


def parse(path):
    txt = open(path).read()
    row = {}
    for key, _ in KEYS:
        m = re.search(r"\| %s[^|]*\| ([0-9.]+) \| ([^|]*)\|" % re.escape(key), txt)
        if m:
            row[key] = "%s %s" % (m.group(1), m.group(2).strip())
    st = re.findall(r"^- (\w+): ([0-9.]+)%", txt, re.M)
    row["top stalls"] = ", ".join("%s %s%%" % s for s in st[:3])
    return row


def main():
    out = sys.argv[1]
    rows = []
    for arg in sys.argv[2:]:
        label, path = arg.rsplit("=", 1)
        rows.append((label, path, parse(path)))
    with open(out, "w") as f:
        f.write("# ncu --set full summary (%s)\n\n" % ", ".join(r[0] for r in rows))
        f.write("| kernel | " + " | ".join(k[1] for k in KEYS) + " | top stalls | source |\n")
        f.write("|---" * (len(KEYS) + 3) + "|\n")
        for label, path, r in rows:
            f.write("| %s | %s | %s | `%s` |\n" % (label, " | ".join(r.get(k[0], "—") for k in KEYS),
                                                  r["top stalls"], path))
    print(open(out).read())


if __name__ == "__main__":
    main()
