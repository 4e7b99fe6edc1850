"""Time assembled-matrix construction on the C5
lattice (16, 64, 64) = 2^16 cells: the symbolic CSR pattern
(sfk_csr_create) once, then the numeric assembly (sfk_assemble_csr: C5
kernel + fused CSR scatter) as the timed step, beside the dense C5 kernel
(A[C][N^6] to HBM) on the same cells.

    python tools/bench_csr.py [--p 1 2 3 4] [--dims 16 64 64]

Roofline of the numeric step: max(F_alg/P64, bytes/BW) with F_alg the C5
per-cell count and bytes = values written once (8 nnz) + col_idx read once
(4 nnz) + row_ptr + coords + dof map.
"""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1711_02473_b200 import compile_kernel, evaluate_batched, runtime, workloads  # noqa
from paper_1711_02473_b200.assembly import (CsrPattern, assemble_csr, insert_csr,  # noqa
                                            lattice_dof_map, lattice_ndofs)
from paper_1711_02473_b200.plan import reference_flops  # noqa

HBM_GBS = 6549.8


def timed(fn, reps, flush):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        torch.cuda._sleep(2_000_000)   # host launch latency off the timed events
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--p", type=int, nargs="*", default=[1, 2, 3, 4])
    ap.add_argument("--dims", type=int, nargs=3, default=[16, 64, 64])
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    p64 = max(runtime.fp64_peak(0.5))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    coords = torch.from_numpy(workloads.lattice_coords(*a.dims)).cuda()
    C = coords.shape[0]
    for p in a.p:
        n3 = (p + 1) ** 3
        g = torch.from_numpy(lattice_dof_map(*a.dims, p)).cuda()
        nd = lattice_ndofs(*a.dims, p)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pat = CsrPattern(g, nd)
        torch.cuda.synchronize()
        t_sym = (time.perf_counter() - t0) * 1e3
        plan = compile_kernel("laplace", "hex", p)
        vals = torch.zeros(pat.nnz, dtype=torch.float64, device="cuda")

        def step():
            vals.zero_()
            assemble_csr(plan, g, coords, pat, values=vals)
        # p >= 5: the DMMA kernel inserts through the entry map only (without
        # one, assemble_csr builds it per call) — no binary-search column
        ms = timed(step, a.reps, flush) if p <= 4 else None
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        emap = pat.entry_map(g)
        torch.cuda.synchronize()
        t_map = (time.perf_counter() - t0) * 1e3

        def step_mapped():
            vals.zero_()
            assemble_csr(plan, g, coords, pat, values=vals, entry_map=emap)
        ms_map = timed(step_mapped, a.reps, flush)
        ms_zero = timed(lambda: vals.zero_(), a.reps, flush)
        dense = torch.empty((C, n3 * n3), dtype=torch.float64, device="cuda")
        ms_dense = timed(lambda: evaluate_batched(plan, {"coords": coords}, out=dense),
                         a.reps, flush)

        # the generic two-pass path every other form uses: cell matrices to
        # HBM, then sfk_csr_insert (entry map) — here on the same matrices
        def step_insert():
            vals.zero_()
            insert_csr(dense, g, pat, values=vals, entry_map=emap)
        ms_insert = timed(step_insert, a.reps, flush)
        del dense, emap
        fl = reference_flops(plan)
        # values written once, col_idx read once, the entry map read once
        nbytes = 12 * pat.nnz + 8 * (nd + 1) + C * (24 * 8 + 4 * n3 + 4 * n3 * n3)
        t_roof = max(fl * C / (p64 * 1e12), nbytes / (HBM_GBS * 1e9)) * 1e3
        rec = {"config": "C5-CSR", "p": p, "cells": C, "ndofs": nd, "nnz": pat.nnz,
               "symbolic_ms": round(t_sym, 2), "entry_map_ms": round(t_map, 2),
               "assemble_search_ms": round(ms, 4) if ms is not None else None, "assemble_ms": round(ms_map, 4),
               "zero_fill_ms": round(ms_zero, 4), "dense_c5_ms": round(ms_dense, 4),
               "insert_ms": round(ms_insert, 4),
               "two_pass_ms": round(ms_dense + ms_insert, 4),
               "nnz_per_s": round(pat.nnz / ms_map * 1e3, 1),
               "bound": "fp64" if fl * C / (p64 * 1e12) >= nbytes / (HBM_GBS * 1e9) else "hbm",
               "roofline_frac": round(t_roof / ms_map, 4), "p64_tflops": round(p64, 2)}
        print(json.dumps(rec), flush=True)
        del pat, vals
        torch.cuda.empty_cache()


if __name__ == "__main__":
    from paper_1711_02473_b200 import runtime as _rt

    print("options from env:", _rt.options_from_env(), file=sys.stderr)
    main()
