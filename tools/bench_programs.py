"""Time the LoopProgram path (generated kernels) on fixture programs, with the
hand-written kernel beside it where one exists.

    python tools/bench_programs.py [--cells N] [key ...]

Inputs: each fixture's seeded cells tiled to N cells (default 2^16) in HBM;
CUDA events around `--reps` launches after warm-up, L2 flushed between.
Prints one JSON line per program.
"""

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1711_02473_b200 import (compile_kernel, evaluate_batched, load_program,  # noqa: E402
                                   program_flops, runtime)

GOLDEN = os.path.join(ROOT, "tests", "golden")
HBM_GBS = 6549.8   # MEASURED_PEAKS.json hbm_gbs
DEFAULT = ["action_laplace_hex_p1", "action_laplace_hex_p2", "action_laplace_hex_p3",
           "action_laplace_hex_p4", "action_laplace_hex_p6", "laplace_hex_p2", "laplace_hex_p3",
           "stokes_momentum_hex_p2", "vector_mass_hex_p2", "weighted_laplace_prism_p2",
           "curl_curl_quad_p2", "action_laplace_quad_p2", "mass_triangle_p2",
           "action_weighted_laplace_hex_p4_colloc"]
HAND = {"action_laplace_hex_p%d" % p: ("action_laplace", "hex", p) for p in range(1, 9)}
HAND.update({"laplace_hex_p%d" % p: ("laplace", "hex", p) for p in range(1, 5)})


def timeit(fn, reps, flush):
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
    ap.add_argument("--cells", type=int, default=1 << 16)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--fma", action="store_true")
    ap.add_argument("--big", action="store_true",
                    help="the p = 5..8 hex Laplace matrices of programs_big.npz (cells capped "
                         "so the output stays under 2 GB)")
    ap.add_argument("keys", nargs="*")
    a = ap.parse_args()
    stem = "programs_big" if a.big else "programs"
    idx = {m["key"]: m for m in json.load(open(os.path.join(GOLDEN, stem + ".json")))}
    z = np.load(os.path.join(GOLDEN, stem + ".npz"))
    if a.big and not a.keys:
        a.keys = list(idx)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    p64 = max(runtime.fp64_peak(0.5))
    for key in a.keys or DEFAULT:
        m = idx[key]
        text = bytes(z[key + "__json"]).decode()
        plan = load_program(text, fma=a.fma)
        cells = a.cells
        if a.big:
            cells = min(cells, max(1, (2 << 30) // (8 * m["return"][1])))
        ins = {}
        for name, size in m["arguments"]:
            v = z["%s__%s" % (key, name)]
            reps = -(-cells // v.shape[0])
            ins[name] = torch.from_numpy(np.tile(v, (reps, 1))[:cells].copy()).cuda()
        out = torch.empty((cells, m["return"][1]), dtype=torch.float64, device="cuda")
        ms = timeit(lambda: evaluate_batched(plan, ins, out=out), a.reps, flush)
        fl = program_flops(text)
        nbytes = 8 * (m["return"][1] + sum(sz for _, sz in m["arguments"]))
        tf = fl * cells / ms * 1e-9
        t_roof = cells * max(fl / (p64 * 1e12), nbytes / (HBM_GBS * 1e9)) * 1e3
        rec = {"key": key, "cells": cells, "ms": round(ms, 5),
               "cells_per_s": round(cells / ms * 1e3, 1), "flops_per_cell_ref": fl,
               "bytes_per_cell": nbytes, "fp64_tflops_ref": round(tf, 3),
               "hbm_gbs": round(nbytes * cells / ms * 1e-6, 1), "p64_tflops": round(p64, 2),
               "bound": "fp64" if fl / (p64 * 1e12) >= nbytes / (HBM_GBS * 1e9) else "hbm",
               "roofline_frac": round(t_roof / ms, 4), "config": plan.config}
        if key in HAND and not key.endswith("colloc") and not a.big:
            hp = compile_kernel(*HAND[key])
            hms = timeit(lambda: evaluate_batched(hp, ins, out=out), a.reps, flush)
            rec["hand_ms"] = round(hms, 5)
            rec["slowdown_vs_hand"] = round(ms / hms, 2)
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    from paper_1711_02473_b200 import runtime as _rt

    print("options from env:", _rt.options_from_env(), file=sys.stderr)
    main()
