#!/usr/bin/env python
"""Summarise ncu captures into profiles/ (run in the CPU container).

    python tools/ncu_summary.py gpurun_out/r01a_prof_p8.ncu-rep KEY [--launches CSV]

Writes profiles/<stem>.md with the key counters of every captured kernel and
merges {KEY: dram bytes per launch} into profiles/ncu_traffic.json (read by
bench.py for roofline.traffic).
"""

from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 inst issued %"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/CTA"),
    ("launch__block_size", "CTA size"),
    ("launch__grid_size", "grid"),
    ("launch__occupancy_limit_registers", "occ. limit (regs)"),
    ("launch__occupancy_limit_shared_mem", "occ. limit (smem)"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem ld bank conflicts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "smem st bank conflicts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return hdr, units, rows[2:]


def stalls(hdr, vals):
    st = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
            try:
                st.append((float(vals[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(v for v, _ in st) or 1.0
    return [(h, v / tot) for v, h in sorted(st, reverse=True)[:8]]


def main():
    rep, key = sys.argv[1], sys.argv[2]
    hdr, units, rows = raw(rep)
    stem = os.path.basename(rep).replace(".ncu-rep", "")
    lines = ["# ncu --set full: %s" % stem, "",
             "Source: `%s` (captured on a B200 via gpurun, `--clock-control none`)." % rep, ""]
    traffic = None
    for vals in rows:
        name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        lines.append("## %s" % name)
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        for m, label in METRICS:
            if m in hdr:
                i = hdr.index(m)
                lines.append("| %s (`%s`) | %s | %s |" % (label, m, vals[i], units[i]))
        rd = hdr.index("dram__bytes_read.sum") if "dram__bytes_read.sum" in hdr else None
        wr = hdr.index("dram__bytes_write.sum") if "dram__bytes_write.sum" in hdr else None
        if rd is not None and wr is not None:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            traffic = (float(vals[rd]) * scale.get(units[rd], 1)
                       + float(vals[wr]) * scale.get(units[wr], 1))
            lines.append("| **traffic per launch** | %.4g | byte |" % traffic)
        lines.append("")
        lines.append("Top stall reasons (share of PC samples):")
        lines.append("")
        for h, f in stalls(hdr, vals):
            lines.append("- %s: %.1f%%" % (h, 100 * f))
        lines.append("")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", stem + ".md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    data = json.load(open(tpath)) if os.path.exists(tpath) else {}
    if traffic is not None:
        data[key] = traffic
    with open(tpath, "w") as f:
        json.dump(data, f, indent=1, sort_keys=True)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
