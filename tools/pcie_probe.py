#!/usr/bin/env python
"""PCIe probe: pinned H2D / D2H bandwidth alone and concurrently, and the
e2e host path (sfk_eval_host) of the C2 action at several chunk sizes."""
import json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1711_02473_b200 import compile_kernel, runtime, workloads

dev = torch.device("cuda", 0)
n = 1 << 30
h = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device=dev)
d2 = torch.empty(n, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best
res = {}
res["h2d_GBs"] = n / t(lambda: d.copy_(h, non_blocking=True)) / 1e9
res["d2h_GBs"] = n / t(lambda: h.copy_(d, non_blocking=True)) / 1e9
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
res["concurrent_total_GBs"] = 2 * n / t(both) / 1e9
for p in (1, 4, 8):
    plan = compile_kernel("action_laplace", "hex", p)
    inp = workloads.c2_inputs(p)
    pc = torch.from_numpy(inp["coords"]).pin_memory()
    pu = torch.from_numpy(inp["w0"]).pin_memory()
    pa = torch.empty_like(pu).pin_memory()
    C = pc.shape[0]
    for chunk in (0, 8192, 32768, 65536):
        dt = t(lambda: runtime.evaluate_host_ptrs(plan, C, pa.data_ptr(), pc.data_ptr(), pu.data_ptr(), None, chunk))
        byt = C * (24 + 2 * (p + 1) ** 3) * 8
        res["p%d_chunk%d" % (p, chunk)] = {"ms": round(dt * 1e3, 2), "GBs": round(byt / dt / 1e9, 1),
                                            "gdofs": round(C * (p + 1) ** 3 / dt / 1e9, 3)}
print(json.dumps(res, indent=1))
