#!/usr/bin/env python
"""Benchmark: Q_p hex Laplace action GDoF/s (fp64) vs degree p on B200.

BASELINE.json metric "Q_p hex Laplace action GDoF/s (fp64) vs degree p; % of
roofline", config C2 (configs[1]): 2^18 jittered trilinear hex cells per GPU,
(p+1)^3 dofs/cell, u ~ U[-1,1], GL (p+1)^3 quadrature, p = 1..8.

A STEP is one application of the action at every degree p = 1..8 over the
whole batch (8 sfk_eval launches, inputs resident in HBM).  value = total
local DoFs processed by all ranks / max-over-ranks device time (GDoF/s).
Weak scaling (default): each rank owns its own 2^18-cell slab of a
(64*N, 64, 64) lattice (cell-range sharding, no data-path collective;
SURVEY.md §8(e)).  `--scaling strong`: the (64, 64, 64) lattice is fixed and
split into ix-slabs over the ranks (SURVEY.md §8(e) asks for both).

Extra keys: per_degree (ms, GDoF/s, cells/s, roofline fraction for every p),
roofline (dominant kernel, vs the FP64 peak measured live), cpu_baseline
(the reference's own emitted C over all host cores, rank 0, N=1), e2e (the
host-buffer C-ABI call sfk_eval_host: H2D + compute + D2H), clocks,
gpu_launches, parity (the device result of EVERY cell against the
reference's own emitted C, rank 0 at N=1), c5 (BASELINE config C5: local
matrices p=1..4 on 2^16 cells per GPU + the NCCL-all-reduced Frobenius
checksum).  `--impl reference` times the reference CPU path alone, on the
full batch.

`--gpus N` with no torchrun environment re-launches itself under
`torch.distributed.run --nproc-per-node N` (one process per GPU); under
torchrun, WORLD_SIZE must equal N.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Q_p hex Laplace action GDoF/s (fp64) vs degree p; % of roofline"
HBM_FALLBACK = 6650.0  # GB/s, B200_PROFILING.md fallback


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None,
                    help="GPUs (one process each); default: WORLD_SIZE or 1")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--degrees", default="1-8")
    ap.add_argument("--lattice", default="64,64,64",
                    help="cells per rank (weak) or in total (strong), nx,ny,nz")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-cells", type=int, default=0,
                    help="cells per degree in the CPU baseline (0 = the whole batch)")
    ap.add_argument("--no-c5", action="store_true", help="skip the C5 checksum leg")
    ap.add_argument("--c5-lattice", default="16,64,64", help="C5 cells per rank, nx,ny,nz")
    ap.add_argument("--backend", choices=["nccl", "gloo"], default="nccl")
    ap.add_argument("--option", action="append", default=[], metavar="NAME=VALUE",
                    help="A/B runs only: libsfk tuning option (runtime.set_option), "
                         "recorded in config.options")
    ap.add_argument("--flush", choices=["clean", "dirty"], default="clean",
                    help="L2 flush between steps: 'dirty' = write 256 MiB (the L2 then "
                         "holds dirty lines the first kernel must write back); 'clean' = "
                         "that write followed by a 256 MiB read, so the L2 holds only "
                         "clean unrelated lines (ncu's cache-control state)")
    ap.add_argument("--shared-device", action="store_true",
                    help="tests only: every rank on cuda:0 (gloo), to exercise the N>1 "
                         "host path on a 1-GPU box; never a scaling number")
    return ap.parse_args()


def _free_port():
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def maybe_relaunch(args):
    """One process per GPU: `python bench.py --gpus N` (no torchrun env)
    re-executes itself under torch.distributed.run; under torchrun the world
    size must match --gpus.  Returns an exit code when it relaunched."""
    env_world = os.environ.get("WORLD_SIZE")
    if args.gpus is None:
        args.gpus = int(env_world or 1)
    if env_world is None:
        if args.gpus > 1 and args.impl == "ours":
            cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                   "--nproc-per-node", str(args.gpus), "--master-addr", "127.0.0.1",
                   "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
            return subprocess.call(cmd)
        return None
    if int(env_world) != args.gpus:
        raise SystemExit("bench.py: --gpus %d but WORLD_SIZE=%s (one process per GPU)"
                         % (args.gpus, env_world))
    return None


SPIN_CYCLES = 2_000_000   # ~1 ms at 1.965 GHz


def degrees_of(s):
    out = []
    for part in s.split(","):
        if "-" in part:
            a, b = part.split("-")
            out.extend(range(int(a), int(b) + 1))
        else:
            out.append(int(part))
    return out


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.15)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------


class L2Flush:
    """Evict the 126 MB L2 between timed steps (outside the timed events).
    'dirty': write a 256 MiB buffer.  'clean' (default): that write, then a
    read of a second 256 MiB buffer, which writes the dirty lines back before
    the step, so the first kernel of the step is not charged for another
    buffer's write-back (the state ncu's cache control gives every kernel)."""

    def __init__(self, dev, mode):
        import torch
        self.mode = mode
        self.wr = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        if mode == "clean":
            self.rd = torch.zeros(32 << 20, dtype=torch.float64, device=dev)
            self.acc = torch.empty((), dtype=torch.float64, device=dev)

    def __call__(self):
        import torch
        self.wr.zero_()
        if self.mode == "clean":
            torch.sum(self.rd, dim=0, out=self.acc)

    def describe(self):
        return ("flushed between steps (256 MiB write + 256 MiB read: no dirty lines)"
                if self.mode == "clean" else "flushed between steps (256 MiB write)")


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _time_ref(ev, plans, inputs, reps):
    """Best-of-reps seconds per degree of evaluator ev over inputs."""
    best = []
    for pl, inp in zip(plans, inputs):
        ev(pl, {"coords": inp["coords"][:64], "w0": inp["w0"][:64]})
        t = 1e30
        for _ in range(reps):
            t0 = time.perf_counter()
            ev(pl, inp)
            t = min(t, time.perf_counter() - t0)
        best.append(t)
    return best


def reference_arm(args):
    """The reference's own CPU path: its emitted C (oracle/_ref) with an
    OpenMP cell loop over all host cores; the oracle port if _ref is absent."""
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import cpu, refc
    from paper_1711_02473_b200 import compile_kernel, workloads

    degs = degrees_of(args.degrees)
    nx, ny, nz = (int(x) for x in args.lattice.split(","))
    sample = min(args.cpu_cells or nx * ny * nz, nx * ny * nz)
    coords = workloads.lattice_coords(nx, ny, nz)[:sample]
    plans = [compile_kernel("action_laplace", "hex", p) for p in degs]
    build_s = None
    if all(refc.key_for(pl) for pl in plans) and os.path.isdir(os.path.join(ROOT, "oracle", "_ref", "src")):
        # compile the reference's emitted C on THIS host (-march=native here)
        build_s = refc.host_build([refc.key_for(pl) for pl in plans])
    kind = "reference" if all(refc.available(pl) for pl in plans) else "port"
    ev = refc.evaluate if kind == "reference" else cpu.evaluate
    inputs = [{"coords": coords, "w0": workloads.uniform_dofs(sample, (p + 1) ** 3)}
              for p in degs]
    # both builds of the reference C: the parity build and
    # the paper's -ffast-math build; the faster one is the reference value
    builds = ["parity"]
    if kind == "reference" and all(refc.available(pl, "fast") for pl in plans):
        builds.append("fast")

    def ev_for(build):
        if kind != "reference":
            return ev
        return lambda pl, inp: refc.evaluate(pl, inp, build=build)
    for _ in range(args.warmup):
        for b in builds:
            for pl, inp in zip(plans, inputs):
                ev_for(b)(pl, {"coords": inp["coords"][:256], "w0": inp["w0"][:256]})
    per_build = {}
    for b in builds:
        per = {p: [] for p in degs}
        for _ in range(args.steps):
            for p, pl, inp in zip(degs, plans, inputs):
                t0 = time.perf_counter()
                ev_for(b)(pl, inp)
                per[p].append(time.perf_counter() - t0)
        per_build[b] = per
    dofs = sum(sample * (p + 1) ** 3 for p in degs)
    totals = {b: sum(min(v) for v in per.values()) for b, per in per_build.items()}
    best_build = min(totals, key=totals.get)
    per = per_build[best_build]
    total_t = totals[best_build]
    value = dofs / total_t / 1e9
    cores = (refc.threads(plans[0]) if kind == "reference" else cpu.num_threads())
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": "GDoF/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total_t * 1e3, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C2 hex Q_p Laplace action, GL (p+1)^3, p=%s" % args.degrees,
                   "cells_per_degree": sample, "sample_of": nx * ny * nz,
                   "same_config": sample == nx * ny * nz},
        "per_degree": [{"p": p, "ms": round(min(per[p]) * 1e3, 4),
                        "gdofs": round(sample * (p + 1) ** 3 / min(per[p]) / 1e9, 6)}
                       for p in degs],
        "cpu_baseline": {"value": round(value, 6), "unit": "GDoF/s", "cores": cores,
                         "kind": kind, "build": best_build, "cpu_model": cpu_model(),
                         "compiled_on_this_host": bool(build_s is not None and all(
                             refc.compiled_on_this_host(pl) for pl in plans)),
                         "host_build_s": None if build_s is None else round(build_s, 1),
                         "by_build": {b: round(dofs / t / 1e9, 6) for b, t in totals.items()},
                         "sample": "%d of %d cells per degree, p=%s, best of %d"
                                   % (sample, nx * ny * nz, args.degrees, args.steps)},
        "e2e": {"value": round(value, 6), "unit": "GDoF/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def parity_err(x, ref):
    """SURVEY.md §8(c) metric: per cell max|y - y_ref| / max|y_ref| (floor
    1e-300), max over cells; NaN cells must be NaN in both."""
    x = np.asarray(x).reshape(ref.shape[0], -1)
    ref = np.asarray(ref).reshape(ref.shape[0], -1)
    worst = 0.0
    for c0 in range(0, ref.shape[0], 1 << 14):
        a, r = x[c0:c0 + (1 << 14)], ref[c0:c0 + (1 << 14)]
        nan_r, nan_a = np.isnan(r).any(axis=1), np.isnan(a).any(axis=1)
        if not np.array_equal(nan_r, nan_a):
            return float("inf")
        ok = ~nan_r
        if ok.any():
            den = np.maximum(np.abs(r[ok]).max(axis=1), 1e-300)
            worst = max(worst, float((np.abs(a[ok] - r[ok]).max(axis=1) / den).max()))
    return worst


def cpu_baseline_leg(degs, coords_all, host_inputs, sample_cells=0, device_out=None):
    """The reference's emitted C on this host, compiled here
    (-march=native = this CPU): parity build and -ffast-math build over all
    cores on the first `sample_cells` cells per degree (0 = the whole batch),
    plus the parity build on 1 thread (smaller sample).  With `device_out`
    ({p: device result}) the parity build's outputs also pin the GPU result
    of every sampled cell: returns (baseline, {p: max rel err})."""
    from oracle import cpu, refc
    from paper_1711_02473_b200 import compile_kernel

    plans = [compile_kernel("action_laplace", "hex", p) for p in degs]
    build_s = None
    if all(refc.key_for(pl) for pl in plans) and os.path.isdir(os.path.join(ROOT, "oracle", "_ref", "src")):
        build_s = refc.host_build([refc.key_for(pl) for pl in plans])
    kind = "reference" if all(refc.available(pl) for pl in plans) else "port"
    n = min(sample_cells or coords_all.shape[0], coords_all.shape[0])
    inputs = [{"coords": coords_all[:n], "w0": host_inputs[p][:n]} for p in degs]
    dofs = sum(n * (p + 1) ** 3 for p in degs)
    out = {"unit": "GDoF/s", "kind": kind, "cpu_model": cpu_model()}
    parity = {}
    sample = ("%s %d cells of the C2 batch per degree p=%d..%d, best of 2"
              % ("all" if n == coords_all.shape[0] else "first", n, degs[0], degs[-1]))

    def timed(ev, pl, inp):
        res, best = None, 1e30
        for _ in range(2):
            t0 = time.perf_counter()
            r = ev(pl, inp)
            best = min(best, time.perf_counter() - t0)
            res = r if res is None else res
        return res, best

    if kind != "reference":
        t = 0.0
        for p, pl, inp in zip(degs, plans, inputs):
            res, tp = timed(cpu.evaluate, pl, inp)
            t += tp
            if device_out is not None:
                parity[p] = parity_err(device_out[p][:n], res)
        out.update(value=round(dofs / t / 1e9, 6), cores=cpu.num_threads(), sample=sample)
        return out, parity
    by = {}
    for b in ("parity", "fast"):
        if not all(refc.available(pl, b) for pl in plans):
            continue
        t = 0.0
        for p, pl, inp in zip(degs, plans, inputs):
            res, tp = timed(lambda pl_, inp_, b=b: refc.evaluate(pl_, inp_, build=b), pl, inp)
            t += tp
            if b == "parity" and device_out is not None:
                parity[p] = parity_err(device_out[p][:n], res)
            del res
        by[b] = round(dofs / t / 1e9, 6)
    best = max(by, key=by.get)
    out.update(value=by[best], build=best, by_build=by, cores=refc.threads(plans[0]),
               sample=sample, compiled_on_this_host=all(refc.compiled_on_this_host(pl)
                                                        for pl in plans),
               host_build_s=None if build_s is None else round(build_s, 1))
    # 1-thread run of the parity build on a smaller sample
    n1 = min(n, 2048)
    in1 = [{"coords": i["coords"][:n1], "w0": i["w0"][:n1]} for i in inputs]
    for pl in plans:
        refc.set_threads(pl, 1)
    try:
        t1 = sum(_time_ref(refc.evaluate, plans, in1, 1))
    finally:
        for pl in plans:
            refc.set_threads(pl, 0)
    out["single_thread"] = {"value": round(sum(n1 * (p + 1) ** 3 for p in degs) / t1 / 1e9, 6),
                            "build": "parity", "sample": "first %d cells per degree" % n1}
    return out, parity


def c5_leg(args, world, rank, dev, stream, flush, p64, hbm):
    """BASELINE config C5: local Laplace matrices (test-major, (p+1)^6 fp64
    per cell) for p = 1..4 on this rank's 2^16-cell slab of a (16*G, 64, 64)
    lattice, timed like C2 (CUDA events, L2 flushed, max over ranks); then
    the Frobenius checksum: device partial sums (sfk_sum_squares) and ONE
    all-reduce of 2 doubles.  Checksum parity: the reference's emitted C
    over the same cells (whole batch at p <= 3, first 4096 cells at p = 4)."""
    import torch
    import torch.distributed as dist

    from oracle import refc
    from paper_1711_02473_b200 import compile_kernel, runtime, workloads
    from paper_1711_02473_b200.parallel import allreduce_sums

    nx, ny, nz = (int(x) for x in args.c5_lattice.split(","))
    coords_np = workloads.lattice_coords(nx * world, ny, nz,
                                         ix_range=(nx * rank, nx * (rank + 1)))
    ncells = coords_np.shape[0]
    coords = torch.from_numpy(coords_np).to(dev)
    lib = runtime.load_library()
    ws = torch.empty(runtime.SUM_WORKSPACE, dtype=torch.float64, device=dev)
    res = {"workload": "C5 hex Laplace local matrices, GL (p+1)^3, p=1..4",
           "cells_per_gpu": ncells, "lattice_per_gpu": [nx, ny, nz], "per_degree": []}
    for p in (1, 2, 3, 4):
        plan = compile_kernel("laplace", "hex", p)
        h = runtime.native_plan(plan)
        A = torch.empty((ncells, plan.return_size), dtype=torch.float64, device=dev)

        def launch():
            runtime._check(lib.sfk_eval(h, ncells, A.data_ptr(), coords.data_ptr(), None, None,
                                        stream.cuda_stream))
        for _ in range(max(args.warmup, 3)):
            launch()
        K = max(1, args.steps)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(K)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for e0, e1 in evs:
            flush()
            torch.cuda._sleep(SPIN_CYCLES)
            e0.record(stream)
            launch()
            e1.record(stream)
        torch.cuda.synchronize()
        ms = sum(e0.elapsed_time(e1) for e0, e1 in evs) / K
        part = runtime.sum_squares(A.reshape(-1), workspace=ws).clone()
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        if args.backend == "gloo":
            t = t.cpu()
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            allreduce_sums(part)
        ms = t.item()
        s2, s1 = part.tolist()
        F, Bb = plan.algorithmic_flops, plan.compulsory_bytes
        tsec = ms * 1e-3
        t_roof = ncells * max(Bb / (hbm * 1e9), F / (p64 * 1e12))
        rec = {"p": p, "ms": round(ms, 5), "cells_per_s": round(world * ncells / tsec, 1),
               "gdofs": round(world * ncells * plan.return_size / tsec / 1e9, 4),
               "fp64_tflops_alg": round(ncells * F / tsec / 1e12, 3),
               "roofline_frac": round(t_roof / tsec, 4),
               "frobenius": math.sqrt(s2), "sum": s1}
        if rank == 0 and world == 1 and not args.no_cpu and refc.available(plan):
            nchk = ncells if p <= 3 else min(ncells, 4096)
            ref = refc.evaluate(plan, {"coords": coords_np[:nchk]})
            got = A[:nchk].cpu().numpy()
            ref2 = float(np.sum(ref * ref))
            mine = runtime.sum_squares(A[:nchk].reshape(-1), workspace=ws)[0].item()
            rec["checksum_parity"] = {"cells": nchk, "rel_err": abs(mine - ref2) / ref2,
                                      "max_rel_err_entries": parity_err(got, ref),
                                      "against": "reference emitted C (oracle/_ref)"}
        res["per_degree"].append(rec)
        del A
    return res


def main():
    args = parse()
    rc = maybe_relaunch(args)
    if rc is not None:
        return rc
    if args.impl == "reference":
        return reference_arm(args)

    import torch
    import torch.distributed as dist

    from paper_1711_02473_b200 import compile_kernel, runtime, workloads

    world, rank, local = dist_env()
    if world > 1:
        ngpu = torch.cuda.device_count()
        if args.shared_device:
            if args.backend != "gloo":
                raise SystemExit("--shared-device needs --backend gloo")
            local = 0
        elif local >= ngpu:
            raise SystemExit("bench.py: rank %d needs GPU %d but only %d are visible"
                             % (rank, local, ngpu))
        torch.cuda.set_device(local)
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    degs = degrees_of(args.degrees)
    nx, ny, nz = (int(x) for x in args.lattice.split(","))

    if args.scaling == "weak":
        # rank r owns the slab ix in [nx*r, nx*(r+1)) of a (nx*world, ny, nz) lattice
        coords_np = workloads.lattice_coords(nx * world, ny, nz,
                                             ix_range=(nx * rank, nx * (rank + 1)))
        ncells = coords_np.shape[0]
        total_cells = world * ncells
        host_u = {p: workloads.uniform_dofs(ncells, (p + 1) ** 3, seed=workloads.SEED_U + rank)
                  for p in degs}
    else:
        # the (nx, ny, nz) lattice is fixed; rank r owns a balanced ix-slab of it
        from paper_1711_02473_b200.parallel import shard_range
        lo, hi = shard_range(nx, rank, world)
        coords_np = workloads.lattice_coords(nx, ny, nz, ix_range=(lo, hi))
        ncells = coords_np.shape[0]
        total_cells = nx * ny * nz
        c0 = lo * ny * nz
        host_u = {p: np.ascontiguousarray(
                      workloads.uniform_dofs(total_cells, (p + 1) ** 3)[c0:c0 + ncells])
                  for p in degs}
    plans = {p: compile_kernel("action_laplace", "hex", p) for p in degs}
    opts = {}
    for kv in args.option:
        k, v = kv.split("=", 1)
        runtime.set_option(k, v if k == "c2_kernel" and not v.lstrip("-").isdigit() else int(v))
        opts[k] = v
    coords = torch.from_numpy(coords_np).to(dev)
    u = {p: torch.from_numpy(host_u[p]).to(dev) for p in degs}
    out = {p: torch.empty_like(u[p]) for p in degs}
    stream = torch.cuda.current_stream(dev)
    lib = runtime.load_library()
    handles = {p: runtime.native_plan(plans[p]) for p in degs}
    flush = L2Flush(dev, args.flush)

    # FP64 peak measured live on this GPU (DFMA chains and DMMA), seconds-long
    dfma, dmma = runtime.fp64_peak(1.0)
    p64 = max(dfma, dmma)

    def launch(p):
        runtime._check(lib.sfk_eval(handles[p], ncells, out[p].data_ptr(), coords.data_ptr(),
                                    u[p].data_ptr(), None, stream.cuda_stream))

    for _ in range(max(args.warmup, 3) if args.warmup > 0 else 0):
        for p in degs:
            launch(p)
    torch.cuda.synchronize()

    K = args.steps
    ev = {p: [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(K)] for p in degs}
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = runtime.launch_count()
    with ClockSampler(dev.index if world == 1 else local) as clk:
        for k in range(K):
            flush()  # L2 flush between steps (outside the timed events)
            # ~1 ms spin on the stream before the step's first event, so the
            # host has enqueued every launch before the GPU reaches them: the
            # per-degree events then time the kernels, not the Python/ctypes
            # launch latency (the p = 1 kernel runs ~23 us; one host launch
            # through ctypes takes ~10-20 us)
            torch.cuda._sleep(SPIN_CYCLES)
            for p in degs:
                e0, e1 = ev[p][k]
                e0.record(stream)
                launch(p)
                e1.record(stream)
        torch.cuda.synchronize()
    gpu_launches = runtime.launch_count() - l0
    if world > 1:
        dist.barrier()
    ms = {p: sorted(e0.elapsed_time(e1) for e0, e1 in ev[p]) for p in degs}
    ms_mean = {p: sum(v) / len(v) for p, v in ms.items()}
    step_ms = sum(ms_mean.values())
    if world > 1:
        t = torch.tensor([step_ms] + [ms_mean[p] for p in degs], dtype=torch.float64,
                         device=dev if args.backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        step_ms = t[0].item()
        ms_mean = {p: t[1 + i].item() for i, p in enumerate(degs)}

    peaks = measured_peaks()
    hbm = peaks.get("hbm_gbs", HBM_FALLBACK)
    total_dofs = sum(total_cells * (p + 1) ** 3 for p in degs)
    value = total_dofs / (step_ms * 1e-3) / 1e9
    per = []
    dom = None
    for p in degs:
        pl = plans[p]
        t = ms_mean[p] * 1e-3
        F = pl.algorithmic_flops
        Bb = pl.compulsory_bytes
        t_roof = ncells * max(Bb / (hbm * 1e9), F / (p64 * 1e12))
        rec = {"p": p, "ms": round(ms_mean[p], 5), "gdofs": round(ncells * (p + 1) ** 3 / t / 1e9, 3),
               # the paper's unique-DoF variant C*p^3/T
               "unique_gdofs": round(ncells * p ** 3 / t / 1e9, 3),
               "cells_per_s": round(ncells / t, 1),
               "fp64_tflops_alg": round(ncells * F / t / 1e12, 3),
               "hbm_gbs": round(ncells * Bb / t / 1e9, 1),
               "roofline_frac": round(t_roof / t, 4),
               "bound": "fp64" if F / (p64 * 1e12) > Bb / (hbm * 1e9) else "hbm"}
        per.append(rec)
        if dom is None or ms_mean[p] > ms_mean[dom["p"]]:
            dom = rec
    domplan = plans[dom["p"]]
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tfile):
        try:
            traffic = json.load(open(tfile)).get("C2_p%d" % dom["p"])
        except ValueError:
            traffic = None
    roofline = {"bound": dom["bound"],
                "achieved": dom["fp64_tflops_alg"] if dom["bound"] == "fp64" else dom["hbm_gbs"],
                "peak": round(p64, 3) if dom["bound"] == "fp64" else hbm,
                "unit": "TFLOP/s" if dom["bound"] == "fp64" else "GB/s",
                "frac": None, "traffic": traffic,
                "kernel": "hex_laplace_action_kernel p=%d" % dom["p"],
                "flops_per_cell": domplan.algorithmic_flops,
                "bytes_per_cell": domplan.compulsory_bytes,
                "peak_source": "measured live: max(DFMA %.2f, DMMA %.2f) TFLOP/s; HBM %s GB/s"
                               % (dfma, dmma, hbm)}
    roofline["frac"] = round(roofline["achieved"] / roofline["peak"], 4)

    line = {"metric": METRIC, "value": round(value, 4), "unit": "GDoF/s", "n_gpus": world,
            "steps": K, "warmup": args.warmup, "ms_per_step": round(step_ms, 5),
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (seeded jittered lattice, u~U[-1,1])",
            "config": {"workload": "C2 hex Q_p Laplace action, GL (p+1)^3, p=%s" % args.degrees,
                       "cells_per_gpu": ncells, "cells_total": total_cells,
                       ("lattice_per_gpu" if args.scaling == "weak" else "lattice_total"):
                           [nx, ny, nz],
                       "parallelism": "cell-range shards x%d" % world,
                       "l2": flush.describe(),
                       **({"options": opts} if opts else {}),
                       "launch": "1 ms GPU spin before each step (host launch latency hidden)"},
            "per_degree": per, "roofline": roofline, "gpu_launches": int(gpu_launches),
            "clocks": clk.summary()}

    # ---- e2e: host buffers through the C-ABI (H2D + compute + D2H) ----------
    if not args.no_e2e:
        d2h = sum(ncells * (p + 1) ** 3 * 8 for p in degs)
        pc = torch.from_numpy(coords_np).pin_memory()
        if world == 1:
            # per step: the coordinates go to the device ONCE (sfk_mesh_upload:
            # every degree evaluates on the same mesh), then every degree's
            # batch is enqueued on the library's staging streams
            # (sfk_eval_host_mesh, async) so the 8 copy pipelines overlap; one
            # wait per step, after which every result is in host memory
            h2d = ncells * 24 * 8 + sum(ncells * (p + 1) ** 3 * 8 for p in degs)
            mesh = runtime.Mesh(ncells)
            pinned = {}
            for p in degs:
                pinned[p] = (torch.from_numpy(host_u[p]).pin_memory(),
                             torch.empty((ncells, (p + 1) ** 3), dtype=torch.float64).pin_memory())
            mesh.upload(pc.data_ptr())
            for p in degs:  # warm-up
                mesh.evaluate_host_ptrs(plans[p], pinned[p][1].data_ptr(), pinned[p][0].data_ptr(),
                                        ncells=min(ncells, 4096))
            t0 = time.perf_counter()
            for _ in range(K):
                mesh.upload(pc.data_ptr())
                for p in degs:
                    mesh.evaluate_host_ptrs(plans[p], pinned[p][1].data_ptr(),
                                            pinned[p][0].data_ptr(), wait=False)
                runtime.host_wait()
            e2e_s = (time.perf_counter() - t0) / K
            ok = all(np.array_equal(pinned[p][1].numpy(), out[p].cpu().numpy()) for p in degs)
            mode = ("sfk_mesh_upload (coordinates once per step) + sfk_eval_host_mesh per "
                    "degree (async, pinned host buffers, all degrees' pipelines overlapped) "
                    "+ sfk_host_wait per step")
            del mesh
        else:
            h2d = sum(ncells * (24 + (p + 1) ** 3) * 8 for p in degs)
            # N > 1: host memory per rank bounded to ONE pinned input and ONE
            # pinned output buffer of the largest degree (8 ranks would
            # otherwise pin ~70 GB); each degree is a synchronous
            # sfk_eval_host call (H2D, kernel and D2H pipelined in chunks),
            # its input staged into the pinned buffer outside the timed calls
            nmax = max((p + 1) ** 3 for p in degs)
            pin_in = torch.empty(ncells * nmax, dtype=torch.float64).pin_memory()
            pin_out = torch.empty(ncells * nmax, dtype=torch.float64).pin_memory()
            e2e_s, ok = 0.0, True
            for p in degs:
                nd = (p + 1) ** 3
                pin_in[:ncells * nd].copy_(torch.from_numpy(host_u[p].reshape(-1)))
                runtime.evaluate_host_ptrs(plans[p], min(ncells, 4096), pin_out.data_ptr(),
                                           pc.data_ptr(), pin_in.data_ptr(), None)
                dist.barrier()
                t0 = time.perf_counter()
                for _ in range(K):
                    runtime.evaluate_host_ptrs(plans[p], ncells, pin_out.data_ptr(),
                                               pc.data_ptr(), pin_in.data_ptr(), None)
                e2e_s += (time.perf_counter() - t0) / K
                ok = ok and np.array_equal(pin_out[:ncells * nd].numpy().reshape(ncells, nd),
                                           out[p].cpu().numpy())
            mode = ("sfk_eval_host per degree (synchronous; one pinned in/out buffer pair "
                    "of the largest degree per rank)")
            tt = torch.tensor([e2e_s], dtype=torch.float64,
                              device=dev if args.backend == "nccl" else "cpu")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_s = tt.item()
        line["e2e"] = {"value": round(total_dofs / e2e_s / 1e9, 4), "unit": "GDoF/s",
                       "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                       "ms_per_step": round(e2e_s * 1e3, 3), "api": mode,
                       "matches_device_path": bool(ok)}

    # ---- CPU baseline + full-batch parity: the reference's emitted C on the
    #      host cores over EVERY cell (rank 0, N=1) ---------------------------
    if rank == 0 and world == 1 and not args.no_cpu:
        dev_out = {p: out[p].cpu().numpy() for p in degs}
        cb, parity = cpu_baseline_leg(degs, coords_np, host_u, args.cpu_cells, dev_out)
        line["cpu_baseline"] = cb
        line["parity"] = {"metric": "per cell max|y-y_ref|/max|y_ref|, max over cells",
                          "tolerance": 1e-12, "against": cb["kind"] == "reference"
                          and "reference emitted C (oracle/_ref, parity build)" or "oracle port",
                          "cells": min(args.cpu_cells or ncells, ncells),
                          "max_rel_err": {str(p): v for p, v in parity.items()},
                          "ok": bool(parity) and max(parity.values()) <= 1e-12}
        del dev_out

    # ---- BASELINE config C5: local matrices + all-reduced checksum ---------
    if not args.no_c5:
        for p in degs:
            out[p] = None
        torch.cuda.empty_cache()
        line["c5"] = c5_leg(args, world, rank, dev, stream, flush, p64, hbm)

    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
