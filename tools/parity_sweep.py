"""Small-batch parity sweep through every kernel family and mode:

    python tools/parity_sweep.py [family ...]
    SFK_C2_KERNEL=v4 python tools/parity_sweep.py c2     # one generation

Families: c2, c3, c4, c5, c1, gs (global operators), csr, lp (generated
kernels: CTA / warp / fused modes).  Every result is compared with the CPU
oracle (or, for the generated kernels, the reference's golden outputs bit for
bit).  odd batch
sizes (partial CTAs, tails) and every mode switch are exercised here instead.
"""

import os
import subprocess
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import cpu  # noqa: E402
from paper_1711_02473_b200 import (REGISTRY, action_form, compile_form, compile_kernel,  # noqa
                                   evaluate_batched, neohookean_residual_form, workloads)


def run(plan, inp, tol=1e-12):
    dev = {k: torch.from_numpy(v).cuda() for k, v in inp.items()}
    out = evaluate_batched(plan, dev).cpu().numpy()
    ref = cpu.evaluate(plan, inp)
    err = float((np.abs(out - ref).max(axis=1) / np.abs(ref).max(axis=1)).max())
    assert err < tol, (plan.name, plan.degree, err)
    return err


def fam_c2():
    gen = os.environ.get("SFK_C2_KERNEL", "auto")
    for p in range(1, 9):
        run(compile_kernel("action_laplace", "hex", p), workloads.c2_inputs(p, dims=(3, 3, 5)))
    print("c2 ok", gen)


def fam_c3():
    for p in (4, 7, 11, 15):
        plan = compile_form(action_form(REGISTRY["weighted_laplace"]), "hex", p, "spectral",
                            "spectral_gll", "collocated-gll")
        run(plan, workloads.c3_inputs(p, dims=(2, 3, 3)))
    print("c3 ok")


def fam_c4():
    for p in (2, 3, 4, 6):
        plan = compile_form(neohookean_residual_form(), "hex", p, quadrature=p + 2)
        inp = workloads.c4_inputs(p, dims=(2, 3, 3))
        inp["w0"] = inp["w0"] * (3.0 / p ** 2)   # keep det F > 0 (BASELINE's draw inverts p >= 5)
        run(plan, inp)
    print("c4 ok")


def fam_c5():
    for p in (1, 2, 3, 4):
        run(compile_kernel("laplace", "hex", p), {"coords": workloads.lattice_coords(2, 2, 3)})
    print("c5 ok")


def fam_c1():
    for p in (1, 3, 6):
        inp = {"coords": workloads.quad_coords(37), "w0": workloads.uniform_dofs(37, (p + 1) ** 2)}
        run(compile_kernel("action_laplace", "quad", p), inp)
    print("c1 ok")


def fam_gs():
    from paper_1711_02473_b200.assembly import GlobalOperator, lattice_dof_map, lattice_ndofs
    dims = (2, 3, 2)
    coords = workloads.lattice_coords(*dims)
    for p in range(1, 9):
        plan = compile_kernel("action_laplace", "hex", p)
        g = lattice_dof_map(*dims, p)
        nd = lattice_ndofs(*dims, p)
        x = np.random.default_rng(1).uniform(-1, 1, nd)
        y = GlobalOperator(plan, torch.from_numpy(g).cuda(), torch.from_numpy(coords).cuda(),
                           nd).apply(torch.from_numpy(x).cuda()).cpu().numpy()
        A = cpu.evaluate(plan, {"coords": coords, "w0": x[g]})
        ref = np.zeros(nd)
        np.add.at(ref, g, A)
        assert np.abs(y - ref).max() <= 1e-12 * np.abs(ref).max(), p
    print("gs ok")


def fam_csr():
    from paper_1711_02473_b200.assembly import (CsrPattern, assemble_csr, lattice_dof_map,
                                                lattice_ndofs)
    dims = (2, 2, 2)
    coords = torch.from_numpy(workloads.lattice_coords(*dims)).cuda()
    for p in (1, 2, 3, 4):
        g = torch.from_numpy(lattice_dof_map(*dims, p)).cuda()
        pat = CsrPattern(g, lattice_ndofs(*dims, p))
        emap = pat.entry_map(g)
        v1 = assemble_csr(compile_kernel("laplace", "hex", p), g, coords, pat)
        v2 = assemble_csr(compile_kernel("laplace", "hex", p), g, coords, pat, entry_map=emap)
        assert (v1 - v2).abs().max().item() <= 1e-12 * v1.abs().max().item(), p
    print("csr ok")


def fam_lp():
    import json

    from oracle.loopprog import run_program
    from paper_1711_02473_b200 import load_program
    z = np.load(os.path.join(ROOT, "tests", "golden", "programs.npz"))
    for key in ("action_laplace_quad_p1", "action_laplace_hex_p2", "laplace_hex_p2",
                "curl_curl_quad_p2", "stokes_momentum_hex_p1_vanilla", "vector_mass_hex_p2"):
        text = bytes(z[key + "__json"]).decode()
        doc = json.loads(text)
        inp = {a: z["%s__%s" % (key, a)] for a, _ in doc["arguments"]}
        out = evaluate_batched(load_program(text),
                               {k: torch.from_numpy(v).cuda() for k, v in inp.items()})
        assert np.array_equal(out.cpu().numpy(), z[key + "__A"]), key
    print("lp ok")


FAMILIES = {"c2": fam_c2, "c3": fam_c3, "c4": fam_c4, "c5": fam_c5, "c1": fam_c1,
            "gs": fam_gs, "csr": fam_csr, "lp": fam_lp}

if __name__ == "__main__":
    from paper_1711_02473_b200 import runtime as _rt

    print("options from env:", _rt.options_from_env(), file=sys.stderr)
    for f in sys.argv[1:] or list(FAMILIES):
        FAMILIES[f]()
    torch.cuda.synchronize()
