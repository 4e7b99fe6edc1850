"""Hex Laplace local matrices beyond the BASELINE degrees (p = 5..8; SURVEY.md
§8(f) row 3 "C5 beyond p = 4").

These matrices ((p+1)^6 entries per cell, 531 441 at p = 8) have two GPU
paths: the hand-written chunked DMMA kernel behind ``compile_kernel("laplace",
"hex", p)`` (csrc/hex_matrix_tcn.cu, dense or fused CSR insertion) and the
generated-kernel path on the reference's own serialized LoopProgram (§8(f)
row 2).  Pinned to fixtures made by the reference itself
(tests/golden/make_programs_big.py: Frobenius norm, sum and every 97th entry
of 2 cells per degree, from the reference's emitted C).

CPU tier: the C oracle (test infrastructure) against those fixtures.
GPU tier: the LoopProgram kernel bit-identical to the reference on the
fixture cells; the hand kernel within 1e-12 of the reference fingerprints and
of the oracle on batches larger than the resident grid (every tuning
variant); both CSR paths against the oracle's matrices summed with np.add.at.
"""

import json
import os
from types import SimpleNamespace

import numpy as np
import pytest

from conftest import GOLDEN
from paper_1711_02473_b200 import compile_kernel, workloads

INDEX = json.load(open(os.path.join(GOLDEN, "programs_big.json")))
KEYS = [m["key"] for m in INDEX]
_Z = np.load(os.path.join(GOLDEN, "programs_big.npz"))


def oracle_plan(p):
    """Tables of the hex Laplace matrix at degree p (the same element and GL
    rule as the action), in the shape oracle/cpu.evaluate reads."""
    a = compile_kernel("action_laplace", "hex", p)
    n = p + 1
    return SimpleNamespace(name="laplace", meta={"cell": "hex"}, n=n, m=a.m, B=a.B, D=a.D,
                           wq=a.wq, Bc=a.Bc, Dc=a.Dc, collocated=False, return_size=n ** 6)


def degree(key):
    return int(key.rsplit("p", 1)[1])


@pytest.mark.parametrize("key", KEYS)
def test_oracle_matches_reference_fingerprint(key):
    from oracle import cpu

    p = degree(key)
    coords = _Z[key + "__coords"]
    A = cpu.evaluate(oracle_plan(p), {"coords": coords})
    fro = np.sqrt(np.sum(A * A, axis=1))
    np.testing.assert_allclose(fro, _Z[key + "__fro"], rtol=1e-12)
    np.testing.assert_allclose(A.sum(axis=1), _Z[key + "__sum"], atol=1e-11 * fro.max())
    samp = A[:, _Z[key + "__idx"]]
    err = np.abs(samp - _Z[key + "__sample"]).max(axis=1) / np.abs(A).max(axis=1)
    assert err.max() < 1e-12, err


def test_fixture_index():
    assert KEYS == ["laplace_hex_p5", "laplace_hex_p6", "laplace_hex_p7", "laplace_hex_p8"]
    for m in INDEX:
        assert m["return"][1] == (degree(m["key"]) + 1) ** 6


@pytest.mark.gpu
@pytest.mark.parametrize("key", KEYS)
def test_gpu_bit_identical_to_reference_fingerprint(cuda, key):
    torch = cuda
    from paper_1711_02473_b200 import evaluate_batched, load_program

    plan = load_program(bytes(_Z[key + "__json"]).decode())
    coords = torch.from_numpy(_Z[key + "__coords"]).cuda()
    A = evaluate_batched(plan, {"coords": coords}).cpu().numpy()
    assert np.array_equal(A[:, _Z[key + "__idx"]], _Z[key + "__sample"])
    np.testing.assert_allclose(np.sqrt(np.sum(A * A, axis=1)), _Z[key + "__fro"], rtol=1e-13)


@pytest.mark.gpu
@pytest.mark.parametrize("p", [5, 6, 7, 8])
def test_gpu_lattice_batch_vs_oracle(cuda, p):
    torch = cuda
    from oracle import cpu
    from paper_1711_02473_b200 import evaluate_batched, load_program

    key = "laplace_hex_p%d" % p
    plan = load_program(bytes(_Z[key + "__json"]).decode())
    coords = workloads.lattice_coords(2, 2, 3 if p <= 6 else 1)
    A = evaluate_batched(plan, {"coords": torch.from_numpy(coords).cuda()}).cpu().numpy()
    ref = cpu.evaluate(oracle_plan(p), {"coords": coords})
    err = (np.abs(A - ref).max(axis=1) / np.abs(ref).max(axis=1)).max()
    assert err < 1e-12, err


@pytest.mark.gpu
def test_gpu_csr_assembly_p5(cuda):
    torch = cuda
    from oracle import cpu
    from paper_1711_02473_b200 import assembly, load_program

    p, (nx, ny, nz) = 5, (2, 2, 1)
    plan = load_program(bytes(_Z["laplace_hex_p5__json"]).decode())
    cmap = assembly.lattice_dof_map(nx, ny, nz, p)
    nd = assembly.lattice_ndofs(nx, ny, nz, p)
    coords = workloads.lattice_coords(nx, ny, nz)
    dm = torch.from_numpy(cmap).cuda()
    pat = assembly.CsrPattern(dm, nd)
    vals = assembly.assemble_csr_from(plan, {"coords": torch.from_numpy(coords).cuda()}, dm, pat)
    dense = pat.matrix(vals).to_dense().cpu().numpy()
    loc = cpu.evaluate(oracle_plan(p), {"coords": coords})
    n3 = (p + 1) ** 3
    ref = np.zeros((nd, nd))
    for c in range(len(cmap)):
        ref[np.ix_(cmap[c], cmap[c])] += loc[c].reshape(n3, n3)
    assert np.abs(dense - ref).max() / np.abs(ref).max() < 1e-12


# ---------------------------------------------------------------------------
# hand-written DMMA kernel (hex_matrix_tcn.cu)

@pytest.mark.gpu
@pytest.mark.parametrize("key", KEYS)
def test_gpu_hand_kernel_vs_reference_fingerprint(cuda, key):
    torch = cuda
    from paper_1711_02473_b200 import evaluate_batched

    p = degree(key)
    plan = compile_kernel("laplace", "hex", p)
    assert (plan.name, plan.return_size) == ("laplace", (p + 1) ** 6)
    coords = torch.from_numpy(_Z[key + "__coords"]).cuda()
    A = evaluate_batched(plan, {"coords": coords}).cpu().numpy()
    fro = np.sqrt(np.sum(A * A, axis=1))
    np.testing.assert_allclose(fro, _Z[key + "__fro"], rtol=1e-12)
    np.testing.assert_allclose(A.sum(axis=1), _Z[key + "__sum"], atol=1e-11 * fro.max())
    samp = A[:, _Z[key + "__idx"]]
    err = np.abs(samp - _Z[key + "__sample"]).max(axis=1) / np.abs(A).max(axis=1)
    assert err.max() < 1e-12, err


@pytest.mark.gpu
@pytest.mark.parametrize("p", [5, 6, 7, 8])
@pytest.mark.parametrize("cfg", [0, 1, 2])
def test_gpu_hand_kernel_vs_oracle(cuda, p, cfg):
    """More cells than the resident grid (persistent CTAs run several cells),
    ragged count, every (iy block, warps) variant."""
    torch = cuda
    from oracle import cpu
    from paper_1711_02473_b200 import evaluate_batched, runtime

    nc = 301 if p <= 6 else 157
    coords = workloads.lattice_coords(4, 8, 10)[:nc]
    plan = compile_kernel("laplace", "hex", p)
    with runtime.options(c5_hi_cfg=cfg):
        A = evaluate_batched(plan, {"coords": torch.from_numpy(coords).cuda()})
        torch.cuda.synchronize()
    A = A.cpu().numpy()
    ref = cpu.evaluate(oracle_plan(p), {"coords": coords})
    err = (np.abs(A - ref).max(axis=1) / np.abs(ref).max(axis=1)).max()
    assert err < 1e-12, err
    # symmetric like the operator
    n3 = (p + 1) ** 3
    M = A[:3].reshape(3, n3, n3)
    assert np.abs(M - M.transpose(0, 2, 1)).max() <= 1e-12 * np.abs(M).max()


@pytest.mark.gpu
@pytest.mark.parametrize("p", [5, 6])
def test_gpu_fused_csr_assembly_high_p(cuda, p):
    """Fused CSR insertion from the DMMA kernel (entry map built by
    assemble_csr) == the oracle's cell matrices summed with np.add.at, and ==
    the two-pass path (dense cell matrices + sfk_csr_insert)."""
    torch = cuda
    from oracle import cpu
    from paper_1711_02473_b200 import assembly, evaluate_batched

    nx, ny, nz = 2, 2, 2
    plan = compile_kernel("laplace", "hex", p)
    cmap = assembly.lattice_dof_map(nx, ny, nz, p)
    nd = assembly.lattice_ndofs(nx, ny, nz, p)
    coords = workloads.lattice_coords(nx, ny, nz)
    dm = torch.from_numpy(cmap).cuda()
    xc = torch.from_numpy(coords).cuda()
    pat = assembly.CsrPattern(dm, nd)
    vals = assembly.assemble_csr(plan, dm, xc, pat)
    dense = pat.matrix(vals).to_dense().cpu().numpy()
    loc = cpu.evaluate(oracle_plan(p), {"coords": coords})
    n3 = (p + 1) ** 3
    ref = np.zeros((nd, nd))
    for c in range(len(cmap)):
        ref[np.ix_(cmap[c], cmap[c])] += loc[c].reshape(n3, n3)
    assert np.abs(dense - ref).max() / np.abs(ref).max() < 1e-12
    two = assembly.insert_csr(evaluate_batched(plan, {"coords": xc}), dm, pat).cpu().numpy()
    assert np.abs(two - vals.cpu().numpy()).max() <= 1e-12 * np.abs(two).max()
