#!/usr/bin/env python
"""Per-config measurements of every BASELINE config (C1..C5) on one B200.

    python tools/bench_configs.py [C1 C2 C3 C4 C5] [--reps 5] [--cpu-cells 4096]

For each config and degree: device time of one sfk_eval over the full
BASELINE batch (CUDA events on the launching stream, L2 flushed between
repetitions, median of --reps), GDoF/s, cells/s, the roofline fraction
(max(bytes/HBM, F_alg/P64) / t, P64 measured live), and the CPU baseline
(the reference's emitted C from oracle/_ref over all host cores, or the
oracle port) on a bounded sample of the same batch.  One JSON line per
(config, degree); the headline C2 line with the full contract is bench.py.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["C1", "C2", "C3", "C4", "C5"],
                    help="C4 also prints C4F lines (the finite displacement draw)")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--cpu-cells", type=int, default=4096)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--p", type=int, nargs="*", default=None, help="only these degrees")
    args = ap.parse_args()

    import torch

    from oracle import cpu, refc
    from paper_1711_02473_b200 import (REGISTRY, action_form, compile_form, compile_kernel,
                                       neohookean_residual_form, runtime, workloads)

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    lib = runtime.load_library()
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush_rd = torch.zeros(32 << 20, dtype=torch.float64, device=dev)
    flush_acc = torch.empty((), dtype=torch.float64, device=dev)
    dfma, dmma = runtime.fp64_peak(0.5)
    p64 = max(dfma, dmma)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        pass
    hbm = peaks.get("hbm_gbs", 6650.0)

    def time_launch(fn):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(args.reps):
            flush.zero_()   # write + read: a clean L2 (bench.py --flush clean)
            torch.sum(flush_rd, dim=0, out=flush_acc)
            torch.cuda._sleep(2_000_000)   # host launch latency off the timed events
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e-3)
        return statistics.median(ts)

    def cpu_time(plan, inputs, n):
        if args.no_cpu:
            return None
        sample = {k: v[:n] for k, v in inputs.items()}
        kind = "reference" if refc.available(plan) else "port"
        ev = refc.evaluate if kind == "reference" else cpu.evaluate
        ev(plan, {k: v[:16] for k, v in sample.items()})
        best = 1e30
        with np.errstate(invalid="ignore"):
            for _ in range(2):
                t0 = time.perf_counter()
                ev(plan, sample)
                best = min(best, time.perf_counter() - t0)
        cores = refc.threads(plan) if kind == "reference" else cpu.num_threads()
        return {"s_per_cell": best / n, "kind": kind, "cores": cores, "sample_cells": n}

    def report(cfg, plan, inputs, dofs_per_cell, fn, extra=None, cpu_plan=None):
        ncells = inputs["coords"].shape[0]
        t = time_launch(fn)
        F = plan.algorithmic_flops
        Bb = plan.compulsory_bytes if extra is None else extra
        t_roof = ncells * max(Bb / (hbm * 1e9), (F or 0) / (p64 * 1e12))
        rec = {"config": cfg, "form": plan.name, "p": plan.degree, "cells": ncells,
               "ms": round(t * 1e3, 5), "gdofs": round(ncells * dofs_per_cell / t / 1e9, 3),
               "cells_per_s": round(ncells / t, 1), "flops_per_cell_alg": F,
               "bytes_per_cell": Bb,
               "fp64_tflops_alg": round(ncells * F / t / 1e12, 3) if F else None,
               "hbm_gbs": round(ncells * Bb / t / 1e9, 1),
               "roofline_frac": round(t_roof / t, 4) if F else None,
               "bound": ("fp64" if F and F / (p64 * 1e12) > Bb / (hbm * 1e9) else "hbm"),
               "p64_tflops": round(p64, 2), "hbm_peak_gbs": hbm}
        c = cpu_time(cpu_plan or plan, inputs, min(args.cpu_cells, ncells))
        if c:
            rec["cpu_baseline"] = {"gdofs": round(dofs_per_cell / c["s_per_cell"] / 1e9, 5),
                                   "cells_per_s": round(1 / c["s_per_cell"], 1),
                                   "cores": c["cores"], "kind": c["kind"],
                                   "sample_cells": c["sample_cells"]}
            rec["speedup_vs_cpu"] = round(c["s_per_cell"] * ncells / t, 1)
        print(json.dumps(rec), flush=True)

    def dev_inputs(inputs):
        return {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in inputs.items()}

    def sfk(plan, d, out):
        h = runtime.native_plan(plan)
        return lambda: runtime._check(lib.sfk_eval(
            h, d["coords"].shape[0], out.data_ptr(), d["coords"].data_ptr(),
            d["w0"].data_ptr() if "w0" in d else None,
            d["w1"].data_ptr() if "w1" in d else None, stream.cuda_stream))

    for cfg in args.configs:
        if cfg == "C1":
            pm = compile_kernel("action_mass", "quad", 3)
            pl = compile_kernel("action_laplace", "quad", 3)
            inp = workloads.c1_inputs()
            d = dev_inputs(inp)
            am = torch.empty((1024, 16), dtype=torch.float64, device=dev)
            al = torch.empty_like(am)
            hm, hl = runtime.native_plan(pm), runtime.native_plan(pl)
            fn = lambda: runtime._check(lib.sfk_eval_pair(  # noqa: E731
                hm, hl, 1024, am.data_ptr(), al.data_ptr(), d["coords"].data_ptr(),
                d["w0"].data_ptr(), stream.cuda_stream))

            class Pair:
                name = "action_mass+action_laplace"
                degree = 3
                algorithmic_flops = 944 + 1872
                compulsory_bytes = 8 * (8 + 16 + 32)
            report("C1", Pair, inp, 16, fn, cpu_plan=pl)
        elif cfg == "C2":
            for p in range(1, 9):
                if args.p and p not in args.p:
                    continue
                plan = compile_kernel("action_laplace", "hex", p)
                inp = workloads.c2_inputs(p)
                d = dev_inputs(inp)
                out = torch.empty_like(d["w0"])
                report("C2", plan, inp, (p + 1) ** 3, sfk(plan, d, out))
                del d, out
        elif cfg == "C2G":
            # global matrix-free operator: fused gather +
            # action + atomic scatter on the (64,64,64) lattice's continuous Q_p
            from paper_1711_02473_b200.assembly import (GlobalOperator, lattice_dof_map,
                                                        lattice_ndofs)
            for p in range(1, 9):
                if args.p and p not in args.p:
                    continue
                plan = compile_kernel("action_laplace", "hex", p)
                dims = (64, 64, 64)
                coords = torch.from_numpy(workloads.lattice_coords(*dims)).to(dev)
                gmap = torch.from_numpy(lattice_dof_map(*dims, p)).to(dev)
                nd = lattice_ndofs(*dims, p)
                op = GlobalOperator(plan, gmap, coords, nd)
                x = torch.rand(nd, dtype=torch.float64, device=dev)
                y = torch.zeros_like(x)
                t = time_launch(lambda: op.apply(x, out=y, accumulate=True))
                C = coords.shape[0]
                # compulsory bytes: coords + map (int32) + x, y (read+write) once
                byt = C * (24 * 8 + 4 * (p + 1) ** 3) + 3 * 8 * nd
                rec = {"config": "C2G", "form": "global action_laplace (gather-scatter)", "p": p,
                       "cells": C, "global_dofs": nd, "ms": round(t * 1e3, 5),
                       "gdofs_local": round(C * (p + 1) ** 3 / t / 1e9, 3),
                       "gdofs_global": round(nd / t / 1e9, 3),
                       "roofline_frac": round(C * max(byt / C / (hbm * 1e9),
                                                      plan.algorithmic_flops / (p64 * 1e12)) / t, 4)}
                print(json.dumps(rec), flush=True)
                del coords, gmap, x, y
        elif cfg in ("C3G", "C4G"):
            # the other fused global operators: C3's weighted collocated Laplace
            # and C4's assembled neo-Hookean residual, on their BASELINE
            # lattices (16, 64, 64)
            from paper_1711_02473_b200.assembly import (GlobalOperator, lattice_dof_map,
                                                        lattice_ndofs, lattice_vector_dof_map)
            dims = (16, 64, 64)
            coords = torch.from_numpy(workloads.lattice_coords(*dims)).to(dev)
            C = coords.shape[0]
            degs = range(4, 17) if cfg == "C3G" else range(2, 7)
            for p in degs:
                if args.p and p not in args.p:
                    continue
                n3 = (p + 1) ** 3
                if cfg == "C3G":
                    plan = compile_form(action_form(REGISTRY["weighted_laplace"]), "hex", p,
                                        "spectral", "spectral_gll", "collocated-gll")
                    gmap = torch.from_numpy(lattice_dof_map(*dims, p)).to(dev)
                    nd = lattice_ndofs(*dims, p)
                    w1 = torch.from_numpy(workloads.c3_inputs(p, dims)["w1"]).to(dev)
                    ndl = n3
                else:
                    plan = compile_form(neohookean_residual_form(), "hex", p, quadrature=p + 2)
                    gmap = torch.from_numpy(lattice_vector_dof_map(*dims, p)).to(dev)
                    nd = 3 * lattice_ndofs(*dims, p)
                    w1 = None
                    ndl = 3 * n3
                op = GlobalOperator(plan, gmap, coords, nd, w1=w1)
                x = (torch.rand(nd, dtype=torch.float64, device=dev) - 0.5) * (0.02 * workloads.H)
                y = torch.zeros_like(x)
                t = time_launch(lambda: op.apply(x, out=y, accumulate=True))
                byt = C * (24 * 8 + 4 * ndl + (8 * n3 if w1 is not None else 0)) + 3 * 8 * nd
                rec = {"config": cfg, "form": "global %s (gather-scatter)" % plan.name, "p": p,
                       "cells": C, "global_dofs": nd, "ms": round(t * 1e3, 5),
                       "gdofs_local": round(C * ndl / t / 1e9, 3),
                       "gdofs_global": round(nd / t / 1e9, 3),
                       "roofline_frac": round(C * max(byt / C / (hbm * 1e9),
                                                      plan.algorithmic_flops / (p64 * 1e12)) / t, 4)}
                print(json.dumps(rec), flush=True)
                del gmap, x, y
            del coords
        elif cfg == "C3":
            spec = action_form(REGISTRY["weighted_laplace"])
            for p in range(4, 17):
                if args.p and p not in args.p:
                    continue
                plan = compile_form(spec, "hex", p, "spectral", "spectral_gll", "collocated-gll")
                inp = workloads.c3_inputs(p)
                d = dev_inputs(inp)
                out = torch.empty_like(d["w0"])
                report("C3", plan, inp, (p + 1) ** 3, sfk(plan, d, out))
                del d, out
        elif cfg == "C4":
            for p in range(2, 7):
                if args.p and p not in args.p:
                    continue
                plan = compile_form(neohookean_residual_form(), "hex", p, quadrature=p + 2)
                inp = workloads.c4_inputs(p)
                d = dev_inputs(inp)
                out = torch.empty_like(d["w0"])
                report("C4", plan, inp, 3 * (p + 1) ** 3, sfk(plan, d, out))
                del d, out
                # C4F: the same batch with the finite draw (amplitude 0.03 h / p^2,
                # tests/test_fullsize_parity.py): BASELINE's draw inverts cells at
                # p >= 5 (all of them at p = 6), whose NaN results take log's
                # special-case path — this line times every point on the finite path
                amp = 0.03 / p ** 2
                inp = dict(inp, w0=workloads.uniform_dofs(inp["coords"].shape[0], 3 * (p + 1) ** 3,
                                                          -amp, amp, seed=99, scale=workloads.H))
                d = dev_inputs(inp)
                out = torch.empty_like(d["w0"])
                report("C4F", plan, inp, 3 * (p + 1) ** 3, sfk(plan, d, out))
                del d, out
        elif cfg == "C5":
            for p in range(1, 5):
                if args.p and p not in args.p:
                    continue
                plan = compile_kernel("laplace", "hex", p)
                inp = workloads.c5_inputs()
                d = dev_inputs(inp)
                nd = (p + 1) ** 3
                out = torch.empty((d["coords"].shape[0], nd * nd), dtype=torch.float64,
                                  device=dev)
                report("C5", plan, inp, nd, sfk(plan, d, out))
                del d, out
        elif cfg == "C5H":
            # C5 beyond the BASELINE degrees: p = 5..8 on
            # the chunked DMMA kernel; (p+1)^6 doubles per cell, so the batch
            # shrinks with p to keep A at 6-9 GB (2^14 .. 2^11 cells)
            for p in range(5, 9):
                if args.p and p not in args.p:
                    continue
                plan = compile_kernel("laplace", "hex", p)
                nx = {5: 4, 6: 2, 7: 1, 8: 1}[p]
                inp = {"coords": workloads.lattice_coords(nx, 64, 64 if p <= 7 else 32)}
                d = dev_inputs(inp)
                nd = (p + 1) ** 3
                out = torch.empty((d["coords"].shape[0], nd * nd), dtype=torch.float64,
                                  device=dev)
                cc = args.cpu_cells
                args.cpu_cells = min(cc, 64)
                report("C5H", plan, inp, nd, sfk(plan, d, out))
                args.cpu_cells = cc
                del d, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    from paper_1711_02473_b200 import runtime as _rt

    print("options from env:", _rt.options_from_env(), file=sys.stderr)
    main()
