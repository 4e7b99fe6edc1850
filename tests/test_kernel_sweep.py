"""tools/kernel_sweep.py: the variant spaces are well-formed and one probe
variant of every family still compiles (nvcc cross-compile, no GPU) — the
probe macros live in the product sources, so a refactor there must not break
the tuning path silently."""
import importlib.util
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _load():
    spec = importlib.util.spec_from_file_location(
        "kernel_sweep", os.path.join(ROOT, "tools", "kernel_sweep.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


KS = _load()
REPRESENTATIVE = {"c3": 9, "c2": 5, "cell": 3, "c4": 6, "c4l": 4, "c5": 3, "c5h": 6, "p1": 2, "c2g": 5, "c3g": 9}


@pytest.mark.parametrize("fam", sorted(REPRESENTATIVE))
def test_variant_space_is_well_formed(fam):
    F = KS.FAMILIES[fam]
    vs = F["variants"](REPRESENTATIVE[fam])
    assert vs, fam
    keys = [tuple(sorted((k, v[k]) for k in F["keys"] if k in v)) for v in vs]
    assert len(set(keys)) == len(keys), "duplicate variants"
    for v in vs:
        assert v["n"] == REPRESENTATIVE[fam]
        assert 32 <= v["threads"] <= 1024 and v["threads"] % 32 == 0
        assert v["smem"] <= KS.SMEM_MAX
        defs = F["defines"](v, "sfk_probe_x")
        assert all(d.startswith("-D") for d in defs)
        assert any(d.endswith("_PROBE_ENTRY=sfk_probe_x") for d in defs)


def test_every_family_has_a_representative():
    assert set(REPRESENTATIVE) == set(KS.FAMILIES)


@pytest.mark.parametrize("fam", sorted(REPRESENTATIVE))
def test_one_probe_variant_compiles(fam, tmp_path):
    from paper_1711_02473_b200 import _build as B

    F = KS.FAMILIES[fam]
    v = F["variants"](REPRESENTATIVE[fam])[0]
    obj = str(tmp_path / "probe.o")
    flags = [f for f in B.NVCC_FLAGS if f != "-lineinfo"]
    r = subprocess.run([B.nvcc()] + flags + F["defines"](v, "sfk_probe_x")
                       + ["-c", os.path.join(B.CSRC, F["src"]), "-o", obj],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
    syms = subprocess.run(["nm", "-g", "--defined-only", obj], capture_output=True, text=True).stdout
    assert " T sfk_probe_x" in syms
