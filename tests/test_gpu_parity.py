"""Parity of the sm_100a kernels (through the C-ABI) with the reference.

Bar (BASELINE.json north_star): relative 1e-12 in fp64 with the SURVEY.md
§8(c) metric — per cell max|y - y_ref| / max|y_ref|, max over cells.
Ground truth: the reference's own outputs (tests/golden) and, for larger
batches, the C oracle (oracle/cpu.py, itself pinned to the golden fixtures in
tests/test_oracle.py).
"""

import os

import numpy as np
import pytest

from conftest import GOLDEN, rel_err
from oracle import cpu
from paper_1711_02473_b200 import (compile_kernel, evaluate_batched, evaluate_host,
                                   launch_count, runtime, sum_squares, workloads)
from paper_1711_02473_b200.errors import ShapeMismatch, UnboundVariable

pytestmark = pytest.mark.gpu
TOL = 1e-12


def _dev(torch, inputs):
    return {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in inputs.items()}


def _run(torch, plan, inputs):
    out = evaluate_batched(plan, _dev(torch, inputs))
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.mark.parametrize("p", range(1, 9))
def test_c2_hex_laplace_action_golden(cuda, p):
    g = np.load(os.path.join(GOLDEN, "c2.npz"))
    plan = compile_kernel("action_laplace", "hex", p)
    inp = {"coords": g["coords"], "w0": g["w0_p%d" % p]}
    assert rel_err(_run(cuda, plan, inp), g["A_p%d" % p]) < TOL


@pytest.mark.parametrize("p", range(1, 9))
@pytest.mark.parametrize("ncells", [1, 7, 509])
def test_c2_hex_laplace_action_vs_oracle(cuda, p, ncells):
    plan = compile_kernel("action_laplace", "hex", p)
    coords = workloads.lattice_coords(8, 8, 8)[:ncells]
    inp = {"coords": coords, "w0": workloads.uniform_dofs(ncells, (p + 1) ** 3)}
    assert rel_err(_run(cuda, plan, inp), cpu.evaluate(plan, inp)) < TOL


@pytest.mark.parametrize("p", [1, 3, 8])
def test_c2_full_size_properties(cuda, p):
    """2^18 cells (BASELINE config C2): sampled oracle parity, linearity and
    the patch test (constants are in the kernel of the Laplacian)."""
    torch = cuda
    plan = compile_kernel("action_laplace", "hex", p)
    inp = workloads.c2_inputs(p)
    dev = _dev(torch, inp)
    A = evaluate_batched(plan, dev)
    rng = np.random.default_rng(0)
    idx = np.sort(rng.choice(inp["coords"].shape[0], 256, replace=False))
    sample = {k: v[idx] for k, v in inp.items()}
    assert rel_err(A[torch.from_numpy(idx).cuda()].cpu().numpy(),
                   cpu.evaluate(plan, sample)) < TOL
    # linearity: A(u + 2v) = A(u) + 2 A(v)
    v = torch.roll(dev["w0"], 1, 0)
    Au = A
    Av = evaluate_batched(plan, {"coords": dev["coords"], "w0": v})
    Auv = evaluate_batched(plan, {"coords": dev["coords"], "w0": dev["w0"] + 2 * v})
    scale = Auv.abs().amax(dim=1)
    err = ((Auv - Au - 2 * Av).abs().amax(dim=1) / scale).max().item()
    assert err < 1e-12
    # patch test: A(1) = 0 relative to A's scale for unit-size data
    ones = torch.ones_like(dev["w0"])
    A1 = evaluate_batched(plan, {"coords": dev["coords"], "w0": ones})
    assert (A1.abs().amax() / Au.abs().amax()).item() < 1e-11


def test_host_path_matches_device_path(cuda):
    torch = cuda
    plan = compile_kernel("action_laplace", "hex", 4)
    inp = workloads.c2_inputs(4, dims=(16, 16, 13))
    dev = _run(torch, plan, inp)
    host = evaluate_host(plan, inp, chunk_cells=1000)   # several pipelined chunks
    assert np.array_equal(dev, host)
    host2 = evaluate_batched(plan, inp)                  # numpy inputs -> host path
    assert np.array_equal(dev, host2)


def test_validation_and_edge_cases(cuda):
    torch = cuda
    plan = compile_kernel("action_laplace", "hex", 2)
    coords = torch.zeros((3, 24), dtype=torch.float64, device="cuda")
    with pytest.raises(UnboundVariable):
        evaluate_batched(plan, {"coords": coords})
    with pytest.raises(ShapeMismatch):
        evaluate_batched(plan, {"coords": coords,
                                "w0": torch.zeros((3, 26), dtype=torch.float64, device="cuda")})
    with pytest.raises(ShapeMismatch):
        evaluate_batched(plan, {"coords": coords,
                                "w0": torch.zeros((4, 27), dtype=torch.float64, device="cuda")})
    # empty batch
    out = evaluate_batched(plan, {"coords": coords[:0],
                                  "w0": torch.zeros((0, 27), dtype=torch.float64, device="cuda")})
    assert out.shape == (0, 27)
    # a single cell passed as flat arrays, like run_kernel
    c = workloads.lattice_coords(1, 1, 1)[0]
    u = workloads.uniform_dofs(1, 27)[0]
    flat = evaluate_batched(plan, {"coords": torch.from_numpy(c).cuda(),
                                   "w0": torch.from_numpy(u).cuda()})
    assert flat.shape == (27,)
    ref = cpu.evaluate(plan, {"coords": c[None], "w0": u[None]})[0]
    assert rel_err(flat.cpu().numpy()[None], ref[None]) < TOL
    # zero dofs -> zero output (SPEC.md action examples)
    z = evaluate_batched(plan, {"coords": torch.from_numpy(c[None]).cuda(),
                                "w0": torch.zeros((1, 27), dtype=torch.float64, device="cuda")})
    assert torch.count_nonzero(z).item() == 0


def test_sum_squares_and_launch_counter(cuda):
    torch = cuda
    x = torch.from_numpy(np.random.default_rng(1).standard_normal(1_000_003)).cuda()
    before = launch_count()
    s = sum_squares(x).cpu().numpy()
    assert launch_count() > before
    xn = x.cpu().numpy()
    assert abs(s[0] - np.dot(xn, xn)) < 1e-12 * np.dot(xn, xn)
    assert abs(s[1] - xn.sum()) < 1e-9
    s2 = sum_squares(x).cpu().numpy()
    assert np.array_equal(s, s2)   # bitwise reproducible


# ---------------------------------------------------------------------------
# C3: GLL-collocated (weighted) Laplace action

from paper_1711_02473_b200 import (REGISTRY, action_form, compile_form,  # noqa: E402
                                   evaluate_batched_pair, neohookean_residual_form)


def _c3_plan(p, weighted=True):
    if weighted:
        return compile_form(action_form(REGISTRY["weighted_laplace"]), "hex", p, "spectral",
                            "spectral_gll", "collocated-gll")
    return compile_kernel("action_laplace", "hex", p, "spectral", "spectral_gll",
                          "collocated-gll")


@pytest.mark.parametrize("p", [1, 2, 4, 6, 8, 12, 16])
def test_c3_golden(cuda, p):
    g = np.load(os.path.join(GOLDEN, "c3.npz"))
    inp = {"coords": g["coords"], "w0": g["w0_p%d" % p], "w1": g["w1_p%d" % p]}
    assert rel_err(_run(cuda, _c3_plan(p), inp), g["A_p%d" % p]) < TOL
    lap = {"coords": g["coords"], "w0": g["w0_p%d" % p]}
    assert rel_err(_run(cuda, _c3_plan(p, False), lap), g["Alap_p%d" % p]) < TOL


@pytest.mark.parametrize("p", range(1, 17))
def test_c3_vs_oracle(cuda, p):
    plan = _c3_plan(p)
    n = p + 1
    nc = 37
    inp = {"coords": workloads.lattice_coords(4, 4, 4)[:nc],
           "w0": workloads.uniform_dofs(nc, n ** 3),
           "w1": workloads.uniform_dofs(nc, n ** 3, 0.5, 2.0, seed=workloads.SEED_KAPPA)}
    assert rel_err(_run(cuda, plan, inp), cpu.evaluate(plan, inp)) < TOL


# ---------------------------------------------------------------------------
# C1: quad Q3 mass + Laplace action (fused pair)


def test_c1_golden_and_fused_pair(cuda):
    torch = cuda
    g = np.load(os.path.join(GOLDEN, "c1.npz"))
    pm = compile_kernel("action_mass", "quad", 3)
    pl = compile_kernel("action_laplace", "quad", 3)
    inp = {"coords": g["coords"], "w0": g["w0"]}
    assert rel_err(_run(torch, pm, inp), g["A_action_mass"]) < TOL
    assert rel_err(_run(torch, pl, inp), g["A_action_laplace"]) < TOL
    full = workloads.c1_inputs()
    am, al = evaluate_batched_pair(pm, pl, _dev(torch, full))
    assert rel_err(am.cpu().numpy(), cpu.evaluate(pm, full)) < TOL
    assert rel_err(al.cpu().numpy(), cpu.evaluate(pl, full)) < TOL
    # fused == separate, bit for bit is not required; parity is
    assert rel_err(am.cpu().numpy(), _run(torch, pm, full)) < 1e-14


@pytest.mark.parametrize("p", range(1, 17))
def test_quad_actions_vs_oracle(cuda, p):
    nc = 45
    inp = {"coords": workloads.quad_coords(nc), "w0": workloads.uniform_dofs(nc, (p + 1) ** 2)}
    for form in ("action_mass", "action_laplace"):
        plan = compile_kernel(form, "quad", p)
        assert rel_err(_run(cuda, plan, inp), cpu.evaluate(plan, inp)) < TOL


# ---------------------------------------------------------------------------
# C5: hex Laplace local matrices


@pytest.mark.parametrize("p", range(1, 5))
def test_c5_golden_and_properties(cuda, p):
    g = np.load(os.path.join(GOLDEN, "c5.npz"))
    plan = compile_kernel("laplace", "hex", p)
    assert rel_err(_run(cuda, plan, {"coords": g["coords"]}), g["A_p%d" % p]) < TOL
    coords = workloads.lattice_coords(4, 4, 3)[:41]
    A = _run(cuda, plan, {"coords": coords})
    assert rel_err(A, cpu.evaluate(plan, {"coords": coords})) < TOL
    nd = (p + 1) ** 3
    M = A.reshape(-1, nd, nd)
    scale = np.abs(M).max()
    assert np.abs(M.sum(axis=2)).max() < 1e-12 * scale           # patch test
    assert np.abs(M - M.transpose(0, 2, 1)).max() < 1e-13 * scale  # symmetry
    # matrix/action consistency
    u = workloads.uniform_dofs(coords.shape[0], nd)
    act = _run(cuda, compile_kernel("action_laplace", "hex", p), {"coords": coords, "w0": u})
    assert rel_err(np.einsum("cij,cj->ci", M, u), act) < 1e-12


@pytest.mark.parametrize("p,opts", [
    (3, {"c5_p3": 1}), (3, {"c5_hi_cfg": 3}), (3, {"c5_hi_cfg": 4}),
    (4, {"c5_p4": 1}), (4, {"c5_p4": 2}), (4, {"c5_hi_cfg": 4}),
])
def test_c5_kernel_variants_vs_oracle(cuda, p, opts):
    """Every selectable C5 kernel at p = 3, 4 (FMA phases, tc4 / tc5, the
    chunked DMMA kernel) on a batch larger than the resident grid."""
    from paper_1711_02473_b200 import runtime

    plan = compile_kernel("laplace", "hex", p)
    coords = workloads.lattice_coords(6, 8, 8)[:379]
    with runtime.options(**opts):
        A = _run(cuda, plan, {"coords": coords})
    assert rel_err(A, cpu.evaluate(plan, {"coords": coords})) < TOL


def test_c5_reference_cell_analytic(cuda):
    g = np.load(os.path.join(GOLDEN, "c5.npz"))
    M1 = np.array([[1 / 3, 1 / 6], [1 / 6, 1 / 3]])
    K1 = np.array([[1.0, -1.0], [-1.0, 1.0]])
    expect = (np.kron(np.kron(K1, M1), M1) + np.kron(np.kron(M1, K1), M1)
              + np.kron(np.kron(M1, M1), K1))
    A = _run(cuda, compile_kernel("laplace", "hex", 1), {"coords": g["ref_coords"]})
    assert np.abs(A.reshape(8, 8) - expect).max() < 1e-14


# ---------------------------------------------------------------------------
# C4: neo-Hookean residual


@pytest.mark.parametrize("p", range(1, 7))
def test_c4_golden(cuda, p):
    g = np.load(os.path.join(GOLDEN, "c4.npz"))
    plan = compile_form(neohookean_residual_form(), "hex", p, quadrature=p + 2)
    for s in ("", "b"):
        inp = {"coords": g["coords"], "w0": g["w0%s_p%d" % (s, p)]}
        ref = g["A%s_p%d" % (s, p)]
        out = _run(cuda, plan, inp)
        assert np.array_equal(np.isnan(out), np.isnan(ref))
        ok = ~np.isnan(ref).any(axis=1)
        if ok.any():
            assert rel_err(out[ok], ref[ok]) < TOL


@pytest.mark.parametrize("p", range(2, 7))
def test_c4_vs_oracle(cuda, p):
    plan = compile_form(neohookean_residual_form(), "hex", p, quadrature=p + 2)
    inp = workloads.c4_inputs(p, dims=(2, 4, 5))
    with np.errstate(invalid="ignore"):
        ref = cpu.evaluate(plan, inp)
    out = _run(cuda, plan, inp)
    assert np.array_equal(np.isnan(out), np.isnan(ref))
    ok = ~np.isnan(ref).any(axis=1)
    if ok.any():
        assert rel_err(out[ok], ref[ok]) < TOL
    # the config's draw inverts elements at p >= 5 (ln J of J <= 0 -> NaN, as
    # in the reference); a smaller displacement keeps every cell finite
    amp = 0.03 / p ** 2
    small = {"coords": inp["coords"],
             "w0": workloads.uniform_dofs(inp["coords"].shape[0], inp["w0"].shape[1],
                                          -amp, amp, seed=7, scale=workloads.H)}
    ref = cpu.evaluate(plan, small)
    assert not np.isnan(ref).any()
    assert rel_err(_run(cuda, plan, small), ref) < TOL


@pytest.mark.parametrize("p", range(2, 7))
def test_c4_component_parallel_kernel(cuda, p):
    """hex_neohookean3.cu (three thread groups, one per displacement
    component; option neo_cfg = 3 forces it, 4 forces the line kernel): same
    operation order as the line kernel, so bit-identical on finite cells, on a
    ragged batch count (cells not a multiple of any CTA batch) and with
    inverted cells (NaN as in the reference); parity with the oracle."""
    plan = compile_form(neohookean_residual_form(), "hex", p, quadrature=p + 2)
    inp = workloads.c4_inputs(p, dims=(3, 5, 7))
    inp = {k: v[:101] for k, v in inp.items()}
    with runtime.options(neo_cfg=4):
        line = _run(cuda, plan, inp)
    with runtime.options(neo_cfg=3):
        comp = _run(cuda, plan, inp)
    assert np.array_equal(np.isnan(comp), np.isnan(line))
    assert np.array_equal(np.nan_to_num(comp), np.nan_to_num(line))
    amp = 0.03 / p ** 2
    small = {"coords": inp["coords"],
             "w0": workloads.uniform_dofs(inp["coords"].shape[0], inp["w0"].shape[1],
                                          -amp, amp, seed=11, scale=workloads.H)}
    ref = cpu.evaluate(plan, small)
    assert not np.isnan(ref).any()
    with runtime.options(neo_cfg=3):
        assert rel_err(_run(cuda, plan, small), ref) < TOL


@pytest.mark.parametrize("cfg", range(1, 8))
def test_c2_p1_kernel_variants(cuda, cfg):
    """The thread-per-cell p = 1 kernel's launch shapes (option p1_cfg = 1..3)
    and its persistent double-buffered forms (4..7: a resident grid looping
    over the batches, more batches than CTAs, ragged last batch) give the
    default kernel's result bit for bit, E-vector and global operator."""
    torch = cuda
    from paper_1711_02473_b200.assembly import GlobalOperator, lattice_dof_map, lattice_ndofs

    plan = compile_kernel("action_laplace", "hex", 1)
    dims = (48, 50, 53)                      # 127200 cells: > resident CTAs x 128
    inp = workloads.c2_inputs(1, dims=dims)
    inp = {k: v[:-37] for k, v in inp.items()}   # ragged
    ref = _run(cuda, plan, inp)
    with runtime.options(p1_cfg=cfg):
        out = _run(cuda, plan, inp)
    assert np.array_equal(out, ref)
    # global operator (atomics: compare to rounding)
    gd = (9, 10, 11)
    coords = torch.from_numpy(workloads.lattice_coords(*gd)).cuda()
    gmap = torch.from_numpy(lattice_dof_map(*gd, 1)).cuda()
    nd = lattice_ndofs(*gd, 1)
    x = torch.from_numpy(np.random.default_rng(5).uniform(-1, 1, nd)).cuda()
    op = GlobalOperator(plan, gmap, coords, nd)
    y0 = op.apply(x).cpu().numpy()
    with runtime.options(p1_cfg=cfg):
        y1 = op.apply(x).cpu().numpy()
    assert np.abs(y1 - y0).max() <= 1e-13 * np.abs(y0).max()


@pytest.mark.parametrize("family,p", [("c3", 4), ("c3", 7), ("c3", 10), ("c3", 11), ("c3", 15),
                                      ("c3", 16), ("c4", 2), ("c4", 3), ("c4", 4), ("c4", 5),
                                      ("c4", 6)])
def test_c3_c4_bitwise_reproducible(cuda, family, p):
    """The swept C3 / C4 kernels (fused x/y contractions, in-place z phases,
    the component-parallel kernel's three-way split of a z-line's points) are
    race-free as far as repetition can tell: five runs on a batch that fills
    the GPU several times over give identical bits."""
    torch = cuda
    if family == "c3":
        plan = compile_form(action_form(REGISTRY["weighted_laplace"]), "hex", p,
                            "spectral", "spectral_gll", "collocated-gll")
        inp = workloads.c3_inputs(p, dims=(8, 16, 16) if p <= 11 else (4, 8, 16))
    else:
        plan = compile_form(neohookean_residual_form(), "hex", p, quadrature=p + 2)
        inp = workloads.c4_inputs(p, dims=(8, 16, 16))
    d = _dev(torch, inp)
    ref = evaluate_batched(plan, d)
    torch.cuda.synchronize()
    for _ in range(4):
        out = evaluate_batched(plan, d)
        torch.cuda.synchronize()
        assert torch.equal(torch.nan_to_num(out), torch.nan_to_num(ref))
        assert torch.equal(torch.isnan(out), torch.isnan(ref))


# ---------------------------------------------------------------------------
# determinism, streams, threads, layouts


def test_bitwise_reproducible_and_stream_concurrency(cuda):
    torch = cuda
    plans = [compile_kernel("action_laplace", "hex", p) for p in (2, 5, 7, 8)]
    ins = [_dev(torch, workloads.c2_inputs(p.degree, dims=(8, 8, 9))) for p in plans]
    ref = [evaluate_batched(p, i) for p, i in zip(plans, ins)]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in plans]
    outs = []
    for p, i, s in zip(plans, ins, streams):
        with torch.cuda.stream(s):
            outs.append(evaluate_batched(p, i))
    torch.cuda.synchronize()
    for a, b in zip(ref, outs):
        assert torch.equal(a, b)      # no atomics anywhere: bitwise identical


def test_host_path_thread_safe(cuda):
    import threading

    plan = compile_kernel("action_laplace", "hex", 3)
    inp = workloads.c2_inputs(3, dims=(8, 8, 8))
    expect = evaluate_host(plan, inp)
    res = [None] * 4

    def work(k):
        res[k] = evaluate_host(plan, inp, chunk_cells=97 + k)

    th = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for r in res:
        assert np.array_equal(r, expect)


def test_device_resident_mesh_equals_host_path(cuda):
    """sfk_mesh: coordinates uploaded once, several degrees evaluated from
    host w0 without re-sending them (async + one wait, and a synchronous
    sub-range) — bit-identical to sfk_eval_host with host coordinates; a
    re-upload of other coordinates is ordered after the earlier work."""
    torch = cuda
    from paper_1711_02473_b200.runtime import Mesh, evaluate_host_ptrs, host_wait

    coords = torch.from_numpy(workloads.lattice_coords(6, 6, 7)).pin_memory()
    nc = coords.shape[0]
    mesh = Mesh(nc)
    mesh.upload(coords.data_ptr())
    outs, ins, plans = {}, {}, {}
    for p in (2, 5, 7):
        plans[p] = compile_kernel("action_laplace", "hex", p)
        ins[p] = torch.from_numpy(workloads.uniform_dofs(nc, (p + 1) ** 3)).pin_memory()
        outs[p] = torch.empty_like(ins[p]).pin_memory()
        mesh.evaluate_host_ptrs(plans[p], outs[p].data_ptr(), ins[p].data_ptr(), wait=False,
                                chunk_cells=37)
    host_wait()
    for p in (2, 5, 7):
        ref = torch.empty_like(ins[p]).pin_memory()
        evaluate_host_ptrs(plans[p], nc, ref.data_ptr(), coords.data_ptr(), ins[p].data_ptr(), None)
        assert torch.equal(outs[p], ref), p
    # a sub-range, synchronous
    part = torch.empty((50, 6 ** 3), dtype=torch.float64).pin_memory()
    w0 = ins[5][100:150].contiguous().pin_memory()
    mesh.evaluate_host_ptrs(plans[5], part.data_ptr(), w0.data_ptr(), first_cell=100, ncells=50)
    assert torch.equal(part, outs[5][100:150])
    # re-upload different coordinates: later evaluations see them
    coords2 = torch.from_numpy(workloads.lattice_coords(6, 6, 7, seed=11)).pin_memory()
    mesh.upload(coords2.data_ptr())
    out2 = torch.empty_like(ins[2]).pin_memory()
    mesh.evaluate_host_ptrs(plans[2], out2.data_ptr(), ins[2].data_ptr())
    ref2 = torch.empty_like(ins[2]).pin_memory()
    evaluate_host_ptrs(plans[2], nc, ref2.data_ptr(), coords2.data_ptr(), ins[2].data_ptr(), None)
    assert torch.equal(out2, ref2)


def test_device_path_concurrent_first_use(cuda):
    """Four host threads create fresh plans and launch on their own streams
    at once, so the per-device launch-shape setup (kernel_shape: the >48 KB
    shared-memory opt-in and the occupancy query, cached under a mutex) runs
    concurrently on first use of each kernel; every result must equal the
    single-threaded one bit for bit (launch state thread safety,
    SPEC.md:580 reentrant kernels)."""
    import threading

    torch = cuda
    degrees = (2, 4, 6, 7, 8, 3, 5, 1)
    ins = {p: _dev(torch, workloads.c2_inputs(p, dims=(5, 6, 7))) for p in degrees}
    res = {}
    errs = []

    def work(k):
        try:
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                for p in degrees[k::4] + degrees[(k + 1) % 4::4]:
                    plan = compile_kernel("action_laplace", "hex", p)
                    out = evaluate_batched(plan, ins[p])
                    stream.synchronize()
                    res[(k, p)] = out
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for (k, p), out in res.items():
        ref = evaluate_batched(compile_kernel("action_laplace", "hex", p), ins[p])
        assert torch.equal(out, ref), (k, p)


def test_non_contiguous_and_offset_inputs(cuda):
    torch = cuda
    plan = compile_kernel("action_laplace", "hex", 4)
    inp = workloads.c2_inputs(4, dims=(4, 4, 5))
    dev = _dev(torch, inp)
    # column-sliced (non-contiguous) coords and an odd cell offset (8-byte
    # aligned only, exercising the cp.async 16-byte phase fix-up)
    wide = torch.zeros((dev["coords"].shape[0], 30), dtype=torch.float64, device="cuda")
    wide[:, 3:27] = dev["coords"]
    off = {"coords": wide[1:, 3:27], "w0": dev["w0"][1:]}
    got = evaluate_batched(plan, off).cpu().numpy()
    ref = cpu.evaluate(plan, {k: v[1:] for k, v in inp.items()})
    assert rel_err(got, ref) < TOL


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8])
def test_c2_every_kernel_generation(cuda, p):
    """Each C2 kernel generation that has an instance for n = p+1 agrees with
    the oracle (the auto selection only changes speed, never results);
    selected in-process through the explicit option API (sfk_set_option)."""
    plan = compile_kernel("action_laplace", "hex", p)
    inp = workloads.c2_inputs(p, dims=(5, 5, 7))
    ref = cpu.evaluate(plan, inp)
    gens = [(g, 0) for g in ("v1", "v2", "v3", "v4", "tc", "cell", "v5", "cellv", "v6", "tc8c")]
    gens += [("v5", g) for g in (1, 2, 3)]
    for gen, g in gens:
        with runtime.options(c2_kernel=runtime.C2_KERNELS[gen], c2_g=g):
            err = rel_err(_run(cuda, plan, inp), ref)
        assert err < TOL, (gen, g, err)


@pytest.mark.parametrize("mode", ["colloc_warps", "neo_cta", "colloc_tc", "colloc_tc8c"])
def test_alternative_kernel_modes(cuda, mode):
    """Kernel modes that are off by default for speed (C3's warp-synchronous
    variant, option colloc_warps; C3's DMMA variant, c3_tc) or on by default
    (C4's warp-synchronous variant; neo_warps = -1 turns it off) agree with
    the oracle too."""
    from paper_1711_02473_b200 import (REGISTRY, action_form, compile_form,
                                       neohookean_residual_form)

    if mode in ("colloc_warps", "colloc_tc", "colloc_tc8c"):
        opts, degrees = (({"colloc_warps": 8}, (1, 2, 3, 4)) if mode == "colloc_warps"
                         else ({"c3_tc": 1}, (7, 11, 15)) if mode == "colloc_tc"
                         else ({"c3_tc": 2}, (7,)))   # one-warp-per-cell DMMA kernel, COL mode
        build = lambda p: compile_form(action_form(REGISTRY["weighted_laplace"]), "hex", p,  # noqa
                                       "spectral", "spectral_gll", "collocated-gll")
        inputs = lambda p: workloads.c3_inputs(p, dims=(3, 5, 7))  # noqa
    else:
        opts, degrees = {"neo_warps": -1}, (1, 2, 3)
        build = lambda p: compile_form(neohookean_residual_form(), "hex", p, quadrature=p + 2)  # noqa
        inputs = lambda p: workloads.c4_inputs(p, dims=(3, 5, 7))  # noqa
    for p in degrees:
        plan, inp = build(p), inputs(p)
        with runtime.options(**opts):
            err = rel_err(_run(cuda, plan, inp), cpu.evaluate(plan, inp))
        assert err < TOL, (mode, p, err)


def test_host_async_overlapping_calls(cuda):
    """sfk_eval_host_async for several degrees back to back (staging buffers
    grow mid-sequence), one sfk_host_wait: every result equals the device
    path bit for bit."""
    torch = cuda
    degs = (1, 3, 2, 5, 4)
    coords = torch.from_numpy(workloads.lattice_coords(9, 10, 11)).pin_memory()
    res = {}
    for p in degs:
        plan = compile_kernel("action_laplace", "hex", p)
        u = torch.from_numpy(workloads.uniform_dofs(coords.shape[0], (p + 1) ** 3)).pin_memory()
        a = torch.empty_like(u).pin_memory()
        runtime.evaluate_host_ptrs(plan, coords.shape[0], a.data_ptr(), coords.data_ptr(),
                                   u.data_ptr(), None, chunk_cells=97, wait=False)
        res[p] = (plan, u, a)
    runtime.host_wait()
    for p, (plan, u, a) in res.items():
        dev = evaluate_batched(plan, {"coords": coords.cuda(), "w0": u.cuda()}).cpu()
        assert torch.equal(a, dev), p


@pytest.mark.parametrize("tag,p", [("gl", p) for p in range(1, 9)] + [("glp2", p) for p in (1, 2, 4)]
                         + [("gll", p) for p in (2, 4, 7)])
def test_hex_mass_action(cuda, tag, p):
    """Hex action_mass (registry forms.py:173, 261-263): the reference's own
    outputs (golden) and the dense numpy restatement on a ragged batch."""
    from oracle import dense
    from test_oracle import mass_plan

    g = np.load(os.path.join(GOLDEN, "mass_hex.npz"))
    plan = mass_plan(tag, p)
    inp = {"coords": g["coords"], "w0": g["w0_%s_p%d" % (tag, p)]}
    assert rel_err(_run(cuda, plan, inp), g["A_%s_p%d" % (tag, p)]) < TOL
    coords = workloads.lattice_coords(3, 3, 5)[:37]
    inp = {"coords": coords, "w0": workloads.uniform_dofs(37, plan.n ** 3)}
    assert rel_err(_run(cuda, plan, inp), dense.evaluate(plan, inp)) < TOL
