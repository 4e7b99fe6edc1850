#!/usr/bin/env python
"""Static SASS instruction mix of the hot kernels in libsfk.so (CPU only).

    python tools/sass_mix.py [OUT.md]

Extracts every cubin from paper_1711_02473_b200/libsfk.so (cuobjdump), and
for each kernel function whose name matches the default instantiations
below counts the instructions that carry the performance claims: FP64 math
(DFMA / DMUL / DADD), tensor-core DMMA, shared-memory traffic (LDS / STS),
asynchronous global->shared staging (LDGSTS; UTMALDG / UBLKCP for TMA /
bulk copies), global loads / stores, barriers, uniform constant loads
(LDCU) and local-memory spills (LDL / STL).  The loops of the line kernels
are fully unrolled, so these static counts are per batch of cells.
"""

from __future__ import annotations

import collections
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1711_02473_b200", "libsfk.so")

# (label, regex on the mangled name) of the kernels the dispatch picks by default
KERNELS = [
    ("C2 p=1 cell", r"hex_laplace_action_p1ILb0E"),
    ("C2 p=2 cellv", r"hex_laplace_action_cellILi3ELi64ELi1ELb0E"),
    ("C2 p=3 v6 (warp-sync)", r"hex_laplace_action_v6ILi4ELi8ELi4ELb0ELb1ELb0E"),
    ("C2 p=4 v6 (ZR)", r"hex_laplace_action_v6ILi5ELi5ELi4ELb1ELb0ELb0E"),
    ("C2 p=5 v6 (ZR)", r"hex_laplace_action_v6ILi6ELi7ELi2ELb1ELb0ELb0E"),
    ("C2 p=6 v6 (ZR)", r"hex_laplace_action_v6ILi7ELi5ELi2ELb1ELb0ELb0E"),
    ("C2 p=7 tc8c (DMMA)", r"hex_laplace_action_tc8cILi3ELb1E"),
    ("C2 p=8 v6 (EG)", r"hex_laplace_action_v6ILi9ELi3ELi2ELb0ELb0ELb1E"),
    ("C2 p=7 tc8 (round 1, DMMA)", r"hex_laplace_action_tc8ILb0E"),
    ("C2 p=8 v5 (round 1)", r"hex_laplace_action_v5ILi9ELi3ELi2ELi2ELb1ELb0E"),
    ("C3 colloc p=8", r"hex_colloc_action_kernelILi9E"),
    ("C4 neo-Hookean p=4", r"hex_neohookean_kernelILi5ELi6E"),
    ("C5 p=3 tc4 (DMMA)", r"hex_laplace_matrix_tc4"),
    ("C5 p=4 tc5 (DMMA)", r"hex_laplace_matrix_tc5"),
]
COLS = ["DFMA", "DMUL", "DADD", "DMMA", "HMMA", "UTCMMA", "LDS", "STS", "LDGSTS", "UTMALDG",
        "UBLKCP", "LDG", "STG", "RED", "BAR", "LDCU", "SHFL", "LDL", "STL"]


def functions(sass):
    cur, body = None, []
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            if cur:
                yield cur, body
            cur, body = m.group(1), []
        elif cur:
            body.append(line)
    if cur:
        yield cur, body


def mix(body):
    c = collections.Counter()
    for line in body:
        m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m:
            op = m.group(1)
            c[op] += 1
            if op.startswith("UTC") and "MMA" in op:
                c["UTCMMA"] += 1
    return c


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "sass_mix.md")
    with tempfile.TemporaryDirectory() as td:
        subprocess.run(["cuobjdump", "-xelf", "all", LIB], cwd=td, check=True,
                       capture_output=True)
        sass = ""
        for f in sorted(os.listdir(td)):
            if f.endswith(".cubin"):
                sass += subprocess.run(["cuobjdump", "-sass", os.path.join(td, f)],
                                       capture_output=True, text=True).stdout
    funcs = list(functions(sass))
    rows = []
    for label, rx in KERNELS:
        hits = [(n, b) for n, b in funcs if re.search(rx, n)]
        if not hits:
            rows.append((label, "(not found)", None))
            continue
        name, body = hits[0]   # first instance matching (the dispatched one above)
        rows.append((label, name, mix(body)))
    lines = ["# Static SASS instruction mix (libsfk.so, sm_100a)", "",
             "`python tools/sass_mix.py` — counts per kernel function (fully unrolled "
             "stages: per batch of cells).  FP64 has no tcgen05 kind, so the tensor path "
             "is DMMA (`mma.sync.m8n8k4.f64`); staging is LDGSTS (cp.async).", "",
             "| kernel | " + " | ".join(COLS) + " | function |",
             "|---|" + "---|" * len(COLS) + "---|"]
    for label, name, c in rows:
        if c is None:
            lines.append("| %s | %s |" % (label, name))
            continue
        lines.append("| %s | %s | `%s` |" % (label, " | ".join(str(c.get(k, 0)) for k in COLS),
                                            name[:60]))
    txt = "\n".join(lines) + "\n"
    with open(out, "w") as f:
        f.write(txt)
    print(txt)


if __name__ == "__main__":
    main()
