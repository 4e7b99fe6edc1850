"""Golden fixtures for the LoopProgram path, made
from the REFERENCE itself.  Run in the build container:

    python tests/golden/make_programs.py            # ~1-2 min, parallel

For every case below the reference compiles the kernel
(``cli.compile_kernel``, cli.py:211-217, or lower_form + run_pipeline +
schedule for non-registry requests), serialises the LoopProgram with its own
``scheduling.serialize_program`` (scheduling.py:465-532) and emits its C
(``scheduling.emit_c``, :617-738).  The C is compiled with the parity flags
of SURVEY.md §8(d) (``-O3 -march=native -ffp-contract=off``) and run over a
batch of seeded cells; a few cells are cross-checked against
``interpreter.run_kernel`` (interpreter.py:279-378).  Frozen into
``programs.npz`` (JSON text + inputs + reference outputs per case) and
``programs.json`` (index).  The emitted C itself is not kept.
"""

from __future__ import annotations

import concurrent.futures as cf
import ctypes
import json
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"

SPECTRAL = "spectral"
# (key, form, cell, degree, mode, variant, quadrature, ncells)
CASES = []
_REG = {
    "mass": ("interval", "quad", "triangle", "hex", "prism"),
    "weighted_mass": ("quad", "triangle", "hex", "prism"),
    "laplace": ("interval", "quad", "triangle", "hex", "prism"),
    "weighted_laplace": ("quad", "hex", "prism"),
    "vector_mass": ("quad", "triangle", "hex", "prism"),
    "stokes_momentum": ("quad", "triangle", "hex", "prism"),
    "rhs_source": ("interval", "quad", "triangle", "hex", "prism"),
    "action_mass": ("quad", "triangle", "hex", "prism"),
    "action_laplace": ("interval", "quad", "triangle", "hex", "prism"),
    "curl_curl": ("quad",),
    "action_curl_curl": ("quad",),
}
for _form, _cells in _REG.items():
    for _cell in _cells:
        for _p in (1, 2):
            CASES.append(("%s_%s_p%d" % (_form, _cell, _p), _form, _cell, _p, SPECTRAL,
                          "equispaced", None, 37))
for _form, _cell, _p in (("laplace", "hex", 1), ("action_laplace", "hex", 2),
                         ("stokes_momentum", "hex", 1), ("stokes_momentum", "prism", 1),
                         ("curl_curl", "quad", 2), ("weighted_laplace", "triangle", 2)):
    for _mode in ("vanilla", "coffee"):
        CASES.append(("%s_%s_p%d_%s" % (_form, _cell, _p, _mode), _form, _cell, _p, _mode,
                      "equispaced", None, 37))
CASES += [
    ("action_laplace_hex_p3", "action_laplace", "hex", 3, SPECTRAL, "equispaced", None, 37),
    ("action_laplace_hex_p4", "action_laplace", "hex", 4, SPECTRAL, "equispaced", None, 21),
    ("action_laplace_hex_p6", "action_laplace", "hex", 6, SPECTRAL, "equispaced", None, 9),
    ("action_laplace_hex_p3_gll5", "action_laplace", "hex", 3, SPECTRAL, "spectral_gll", "5", 37),
    ("action_laplace_hex_p3_colloc", "action_laplace", "hex", 3, SPECTRAL, "spectral_gll",
     "collocated-gll", 37),
    ("laplace_hex_p3", "laplace", "hex", 3, SPECTRAL, "equispaced", None, 5),
    ("laplace_hex_p4", "laplace", "hex", 4, SPECTRAL, "equispaced", None, 3),
    ("action_weighted_laplace_hex_p4_colloc", "weighted_laplace@action", "hex", 4, SPECTRAL,
     "spectral_gll", "collocated-gll", 21),
]

CFLAGS = ["-O3", "-march=native", "-ffp-contract=off", "-fPIC", "-shared"]


def _nodes(cell):
    """Vertex positions in the coordinate element's node order."""
    from sumfact import elements
    if cell == "interval":
        return np.array([[0.0], [1.0]])
    if cell == "quad":
        return np.array([[a, b] for a in (0.0, 1.0) for b in (0.0, 1.0)])
    if cell == "hex":
        return np.array([[a, b, c] for a in (0.0, 1.0) for b in (0.0, 1.0) for c in (0.0, 1.0)])
    tri = np.array(elements.triangle_lagrange(1).nodes, dtype=float)
    if cell == "triangle":
        return tri
    if cell == "prism":
        return np.array([[t[0], t[1], z] for t in tri for z in (0.0, 1.0)])
    raise ValueError(cell)


def _program(form, cell, degree, mode, variant, quad):
    from sumfact import cli, forms, passes, scheduling
    if form.endswith("@action"):
        spec = forms.action_form(forms.REGISTRY[form.split("@")[0]])
        el = forms.form_element(spec, cell, degree, variant)
        ce = [forms.coefficient_element(spec, fam, cell, degree, variant)
              for (_o, fam) in spec.coefficient_slots]
        rule = forms.default_quadrature(cell, degree, collocated_gll=(quad == "collocated-gll"))
        k = forms.lower_form(spec, el, rule, cell, coeff_elements=ce,
                             meta={"mode": mode, "variant": variant})
        return scheduling.schedule(passes.run_pipeline(k, mode))
    return cli.compile_kernel(form, cell, degree, mode, variant, quad)


def _one(case):
    key, form, cell, degree, mode, variant, quad, ncells = case
    if REF not in sys.path:
        sys.path.insert(0, REF)
    from sumfact import interpreter, scheduling
    prog = _program(form, cell, degree, mode, variant, quad)
    text = scheduling.serialize_program(prog)
    src = scheduling.emit_c(prog)
    rng = np.random.default_rng(sum(map(ord, key)) * 7919 + degree)
    # keep the fixture small: at most ~20k output doubles per case
    ncells = int(min(ncells, max(2, 20000 // prog.return_buffer[1])))
    inputs = {}
    nodes = _nodes(cell)
    for name, size in prog.arguments:
        if name == "coords":
            x = nodes[None] + rng.uniform(-0.1, 0.1, size=(ncells,) + nodes.shape)
            inputs[name] = np.ascontiguousarray(x.reshape(ncells, -1))
            assert inputs[name].shape[1] == size, (key, size, nodes.shape)
        else:
            inputs[name] = rng.uniform(-1.0, 1.0, size=(ncells, size))
    # compile the reference's C with a cell loop and run it
    args = [a for a, _ in prog.arguments]
    call = ", ".join(["A + c * %dLL" % prog.return_buffer[1]]
                     + ["%s + c * %dLL" % (a, s) for a, s in prog.arguments])
    drv = "\nvoid run_cells(long long n, double *A, %s) {\n  for (long long c = 0; c < n; ++c) %s(%s);\n}\n" % (
        ", ".join("const double *%s" % a for a in args), prog.name, call)
    with tempfile.TemporaryDirectory() as td:
        cpath = os.path.join(td, "k.c")
        with open(cpath, "w") as fh:
            fh.write(src + drv)
        so = os.path.join(td, "k.so")
        subprocess.run(["gcc"] + CFLAGS + ["-o", so, cpath, "-lm"], check=True)
        lib = ctypes.CDLL(so)
        A = np.zeros((ncells, prog.return_buffer[1]))
        dp = ctypes.POINTER(ctypes.c_double)
        lib.run_cells(ctypes.c_longlong(ncells), A.ctypes.data_as(dp),
                      *[inputs[a].ctypes.data_as(dp) for a in args])
    # cross-check the reference interpreter on two cells
    for c in (0, ncells - 1):
        ref = interpreter.run_kernel(prog, {a: inputs[a][c] for a in args})
        scale = max(np.max(np.abs(ref)), 1e-300)
        assert np.max(np.abs(ref - A[c])) / scale < 1e-12, key
    flags = {"transcendental": any(t in text for t in ('"call","sqrt"', '"call","sin"',
                                                       '"call","cos"', '"call","exp"',
                                                       '"call","ln"', '"call","tan"', '"pow"'))}
    meta = {"key": key, "form": form, "cell": cell, "degree": degree, "mode": mode,
            "variant": variant, "quadrature": quad, "ncells": ncells, "name": prog.name,
            "return": list(prog.return_buffer), "arguments": [list(a) for a in prog.arguments],
            "flops": scheduling.count_flops(prog).total_flops, **flags}
    return key, text, inputs, A, meta


def main():
    arrays = {}
    index = []
    with cf.ProcessPoolExecutor(max_workers=os.cpu_count()) as ex:
        for key, text, inputs, A, meta in ex.map(_one, CASES):
            arrays[key + "__json"] = np.frombuffer(text.encode(), dtype=np.uint8)
            for a, v in inputs.items():
                arrays["%s__%s" % (key, a)] = v
            arrays[key + "__A"] = A
            index.append(meta)
            print("%-45s A%-8s json %6d B" % (key, A.shape, len(text)), flush=True)
    np.savez_compressed(os.path.join(HERE, "programs.npz"), **arrays)
    with open(os.path.join(HERE, "programs.json"), "w") as fh:
        json.dump(index, fh, indent=1)


if __name__ == "__main__":
    main()
