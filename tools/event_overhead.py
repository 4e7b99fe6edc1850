"""How much of a short kernel's event-timed duration is the kernel?

For the C2 action at the given degrees, on a (64,64,64) lattice:
  single_dirty  one launch between two events after a 256 MiB write (dirty L2)
  single_clean  one launch between two events after write + 256 MiB read
  b2b           R launches back to back between ONE event pair, / R
  empty         an event pair around a 1-cycle torch.cuda._sleep
Prints one JSON line per degree.  python tools/event_overhead.py 1,2,3
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1711_02473_b200 import compile_kernel, runtime, workloads  # noqa: E402


def main():
    degs = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,2").split(",")]
    dev = torch.device("cuda", 0)
    lib = runtime.load_library()
    s = torch.cuda.current_stream()
    coords = torch.from_numpy(workloads.lattice_coords(64, 64, 64)).to(dev)
    n = coords.shape[0]
    wr = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    rd = torch.zeros(32 << 20, dtype=torch.float64, device=dev)
    acc = torch.empty((), dtype=torch.float64, device=dev)
    K, R = 20, 20

    def ev():
        return torch.cuda.Event(enable_timing=True)

    for p in degs:
        plan = compile_kernel("action_laplace", "hex", p)
        h = runtime.native_plan(plan)
        u = torch.rand((n, (p + 1) ** 3), dtype=torch.float64, device=dev)
        out = torch.empty_like(u)

        def launch():
            runtime._check(lib.sfk_eval(h, n, out.data_ptr(), coords.data_ptr(),
                                        u.data_ptr(), None, s.cuda_stream))
        for _ in range(5):
            launch()
        res = {"p": p}
        for mode in ("dirty", "clean"):
            ts = []
            for _ in range(K):
                wr.zero_()
                if mode == "clean":
                    torch.sum(rd, dim=0, out=acc)
                torch.cuda._sleep(2_000_000)
                a, b = ev(), ev()
                a.record(s)
                launch()
                b.record(s)
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            ts.sort()
            res["single_%s_ms" % mode] = round(sum(ts) / K, 5)
            res["single_%s_min_ms" % mode] = round(ts[0], 5)
        wr.zero_()
        torch.sum(rd, dim=0, out=acc)
        torch.cuda._sleep(2_000_000)
        a, b = ev(), ev()
        a.record(s)
        for _ in range(R):
            launch()
        b.record(s)
        torch.cuda.synchronize()
        res["b2b_ms"] = round(a.elapsed_time(b) / R, 5)
        ts = []
        for _ in range(K):
            torch.cuda._sleep(2_000_000)
            a, b = ev(), ev()
            a.record(s)
            torch.cuda._sleep(1)
            b.record(s)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        res["empty_ms"] = round(sum(ts) / K, 5)
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
