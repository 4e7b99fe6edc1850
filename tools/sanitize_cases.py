"""Small launches of every kernel family and mode, for compute-sanitizer.

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py [FAMILY ...]

Families: c1 c2 c3 c4 c5 mass c2g csr lp.  Each case runs one small ragged
batch (a few CTAs, last batch partial) through the C ABI and checks the
result against the C oracle (so a sanitizer run is also a parity run).
Prints one line per case; exit status 1 on a parity failure.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import cpu  # noqa: E402  (checker only)
from paper_1711_02473_b200 import (REGISTRY, action_form, compile_form,  # noqa: E402
                                   compile_kernel, neohookean_residual_form, runtime,
                                   workloads)
from paper_1711_02473_b200 import assembly  # noqa: E402

DEV = torch.device("cuda", 0)
FAIL = []


def err(got, ref):
    fin = np.isfinite(ref)
    d = np.where(fin, np.abs(got - ref), 0.0)
    s = np.where(fin, np.abs(ref), 0.0).max(axis=1)
    return float((d.max(axis=1) / np.maximum(s, 1e-300)).max()) if len(ref) else 0.0


def run(label, plan, inp, tol=1e-12, ref=None):
    dev = {k: torch.from_numpy(v).to(DEV) for k, v in inp.items()}
    out = runtime.evaluate_batched(plan, dev)
    torch.cuda.synchronize()
    e = err(out.cpu().numpy(), cpu.evaluate(plan, inp) if ref is None else ref)
    ok = e < tol
    print("%-40s cells %4d  rel err %.2e  %s" % (label, inp["coords"].shape[0], e,
                                                  "ok" if ok else "FAIL"), flush=True)
    if not ok:
        FAIL.append(label)


def c1():
    for kind in ("action_mass", "action_laplace"):
        for p in (1, 3, 8):
            pl = compile_kernel(kind, "quad", p)
            inp = {"coords": workloads.quad_coords(45), "w0": workloads.uniform_dofs(45, (p + 1) ** 2)}
            run("C1 %s quad p=%d" % (kind, p), pl, inp)


def c2():
    gens = ["v1", "v2", "v3", "v4", "tc", "cell", "v5", "cellv", "v6", "tc8c"]
    for p in range(1, 9):
        pl = compile_kernel("action_laplace", "hex", p)
        inp = workloads.c2_inputs(p, dims=(3, 3, 5))
        for g in gens:
            with runtime.options(c2_kernel=runtime.C2_KERNELS[g]):
                run("C2 p=%d %s" % (p, g), pl, inp)


def c3():
    for p in (1, 4, 8, 12, 16):
        pl = compile_form(action_form(REGISTRY["weighted_laplace"]), "hex", p, "spectral",
                          "spectral_gll", "collocated-gll")
        run("C3 p=%d" % p, pl, workloads.c3_inputs(p, dims=(3, 3, 5)))
    for opt in ({"colloc_warps": 8}, {"c3_tc": 1}):
        for p in (3, 7):
            pl = compile_form(action_form(REGISTRY["weighted_laplace"]), "hex", p, "spectral",
                              "spectral_gll", "collocated-gll")
            with runtime.options(**opt):
                run("C3 p=%d %s" % (p, opt), pl, workloads.c3_inputs(p, dims=(3, 3, 5)))


def c4():
    for p in range(1, 7):
        pl = compile_form(neohookean_residual_form(), "hex", p, quadrature=p + 2)
        inp = workloads.c4_inputs(p, dims=(3, 3, 5))
        inp["w0"] = inp["w0"] * (3.0 / (p * p))   # finite draw (no inverted cells)
        run("C4 p=%d" % p, pl, inp)
        with runtime.options(neo_warps=-1):
            run("C4 p=%d neo_cta" % p, pl, inp)


def c5():
    for p in (1, 2, 3, 4):
        pl = compile_kernel("laplace", "hex", p)
        run("C5 p=%d" % p, pl, {"coords": workloads.lattice_coords(3, 3, 5)})


def mass():
    for p in (1, 3, 5):
        pl = compile_kernel("action_mass", "hex", p)
        from oracle import dense
        inp = workloads.c2_inputs(p, dims=(3, 3, 5))
        run("mass hex p=%d" % p, pl, inp, ref=dense.evaluate(pl, inp))


def c2g():
    for p in range(1, 9):
        pl = compile_kernel("action_laplace", "hex", p)
        nx, ny, nz = 3, 3, 5
        cmap = assembly.lattice_dof_map(nx, ny, nz, p)
        nd = assembly.lattice_ndofs(nx, ny, nz, p)
        coords = workloads.lattice_coords(nx, ny, nz)
        op = assembly.GlobalOperator(pl, torch.from_numpy(cmap).to(DEV),
                                     torch.from_numpy(coords).to(DEV), nd)
        x = np.random.default_rng(p).uniform(-1, 1, nd)
        y = op.apply(torch.from_numpy(x).to(DEV)).cpu().numpy()
        loc = cpu.evaluate(pl, {"coords": coords, "w0": x[cmap]})
        ref = np.zeros(nd)
        np.add.at(ref, cmap, loc)
        e = float(np.abs(y - ref).max() / np.abs(ref).max())
        ok = e < 1e-12
        print("%-40s cells %4d  rel err %.2e  %s" % ("C2G p=%d" % p, len(cmap), e,
                                                      "ok" if ok else "FAIL"), flush=True)
        if not ok:
            FAIL.append("C2G p=%d" % p)


def csr():
    for p in (1, 2, 3, 4):
        pl = compile_kernel("laplace", "hex", p)
        nx, ny, nz = 2, 3, 3
        cmap = assembly.lattice_dof_map(nx, ny, nz, p)
        nd = assembly.lattice_ndofs(nx, ny, nz, p)
        coords = workloads.lattice_coords(nx, ny, nz)
        dm = torch.from_numpy(cmap).to(DEV)
        pat = assembly.CsrPattern(dm, nd)
        vals = assembly.assemble_csr(pl, dm, torch.from_numpy(coords).to(DEV), pat)
        torch.cuda.synchronize()
        dense = pat.matrix(vals).to_dense().cpu().numpy()
        loc = cpu.evaluate(pl, {"coords": coords})
        n3 = (p + 1) ** 3
        ref = np.zeros((nd, nd))
        for c in range(len(cmap)):
            ref[np.ix_(cmap[c], cmap[c])] += loc[c].reshape(n3, n3)
        e = float(np.abs(dense - ref).max() / np.abs(ref).max())
        ok = e < 1e-12
        print("%-40s cells %4d  rel err %.2e  %s" % ("CSR p=%d" % p, len(cmap), e,
                                                      "ok" if ok else "FAIL"), flush=True)
        if not ok:
            FAIL.append("CSR p=%d" % p)


def lp():
    import json
    from paper_1711_02473_b200 import load_program
    index = json.load(open(os.path.join(ROOT, "tests", "golden", "programs.json")))
    data = np.load(os.path.join(ROOT, "tests", "golden", "programs.npz"))
    keys = ["action_laplace_hex_p3", "laplace_hex_p2", "curl_curl_quad_p2_coffee",
            "stokes_momentum_hex_p1_vanilla", "weighted_laplace_prism_p2", "mass_triangle_p2"]
    meta = {m["key"]: m for m in index}
    for key in keys:
        if key not in meta:
            continue
        plan = load_program(bytes(data[key + "__json"]).decode())
        ins = {a: data["%s__%s" % (key, a)] for a, _ in meta[key]["arguments"]}
        out = runtime.evaluate_batched(plan, {k: torch.from_numpy(v).to(DEV) for k, v in ins.items()})
        torch.cuda.synchronize()
        ref = data[key + "__A"]
        e = float(np.abs(out.cpu().numpy() - ref).max() / max(np.abs(ref).max(), 1e-300))
        ok = e <= 1e-13
        print("%-40s rel err %.2e  %s" % ("LP " + key, e, "ok" if ok else "FAIL"), flush=True)
        if not ok:
            FAIL.append("LP " + key)


FAMILIES = {"c1": c1, "c2": c2, "c3": c3, "c4": c4, "c5": c5, "mass": mass, "c2g": c2g,
            "csr": csr, "lp": lp}

if __name__ == "__main__":
    fams = sys.argv[1:] or list(FAMILIES)
    for f in fams:
        try:
            FAMILIES[f]()
        except Exception as e:  # report and continue: a sanitizer run covers every family
            print("%s: ERROR %r" % (f, e), flush=True)
            FAIL.append(f)
    print("FAILED: %s" % FAIL if FAIL else "all cases ok")
    sys.exit(1 if FAIL else 0)
