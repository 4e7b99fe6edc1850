"""LoopProgram path: the reference's serialized
LoopProgram -> generated sm_100a kernel (libsfk, NVRTC) -> batched cells.

Pins (CPU): the numpy oracle (oracle/loopprog.py, a restatement of
interpreter.run_kernel) reproduces the reference's emitted C bit-for-bit on
every fixture of tests/golden/programs.npz (made by make_programs.py from the
reference itself); libsfk parses and generates every fixture and NVRTC
compiles a sample.  Parity (GPU): every fixture bit-identical to the
reference's -ffp-contract=off C, the FMA build within 1e-12, and a lattice
batch against the hand-written kernels.
"""

import ctypes
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, rel_err
from oracle.loopprog import program_iterations, run_program
from paper_1711_02473_b200 import (compile_kernel, evaluate_batched, load_program,
                                   program_flops, runtime)
from paper_1711_02473_b200 import workloads
from paper_1711_02473_b200.errors import NativeError

INDEX = json.load(open(os.path.join(GOLDEN, "programs.json")))
KEYS = [m["key"] for m in INDEX]
META = {m["key"]: m for m in INDEX}
_Z = None


def fixture(key):
    global _Z
    if _Z is None:
        _Z = np.load(os.path.join(GOLDEN, "programs.npz"))
    m = META[key]
    text = bytes(_Z[key + "__json"]).decode()
    inputs = {a: _Z["%s__%s" % (key, a)] for a, _ in m["arguments"]}
    return text, inputs, _Z[key + "__A"]


# ---------------------------------------------------------------------------
# CPU tier


def test_fixture_index_covers_every_registry_form_and_cell():
    forms = {(m["form"], m["cell"]) for m in INDEX}
    assert ("stokes_momentum", "prism") in forms and ("curl_curl", "quad") in forms
    assert {m["mode"] for m in INDEX} == {"spectral", "vanilla", "coffee"}
    assert {m["cell"] for m in INDEX} == {"interval", "quad", "triangle", "hex", "prism"}


@pytest.mark.parametrize("key", KEYS)
def test_oracle_matches_reference_bitwise(key):
    text, inputs, ref = fixture(key)
    if program_iterations(text) > 300000:
        pytest.skip("large program")
    out = run_program(text, inputs)
    assert np.array_equal(out, ref), rel_err(out, ref)


def test_generate_every_fixture_without_jit():
    for key in KEYS:
        text, _, _ = fixture(key)
        plan = load_program(text, jit=False)
        m = META[key]
        assert plan.name == m["name"]
        assert list(plan.return_buffer) == m["return"]
        assert [list(a) for a in plan.arguments] == m["arguments"]
        cfg = plan.config
        assert cfg["cells_per_block"] in (1, 2, 4, 8, 16, 32)
        assert cfg["threads"] % 32 == 0 and cfg["threads"] <= 512
        assert cfg["cubin_bytes"] == 0
        if cfg["global_scratch"]:
            assert cfg["smem_bytes"] <= 64 * 1024 + 16
        else:
            assert cfg["smem_bytes"] <= 227 * 1024
        src = plan.cuda_source
        assert plan.entry in src and "__global__" in src
        # deterministic generation
        assert load_program(text, jit=False).cuda_source == src


def test_program_flops_equal_reference_count_flops():
    for key in KEYS:
        text, _, _ = fixture(key)
        assert program_flops(text) == META[key]["flops"], key


def test_imperfect_nests_run_thread_per_cell():
    text, _, _ = fixture("stokes_momentum_hex_p1_vanilla")
    cfg = load_program(text, jit=False).config
    assert cfg["serial_phases"] >= 1
    text, _, _ = fixture("laplace_hex_p4")
    assert load_program(text, jit=False).config["global_scratch"] == 1


def _nvrtc_available():
    try:
        ctypes.CDLL("libnvrtc.so.12")
        return True
    except OSError:
        return os.path.exists("/usr/local/cuda/lib64/libnvrtc.so.12")


@pytest.mark.skipif(not _nvrtc_available(), reason="no NVRTC")
@pytest.mark.parametrize("key", ["action_laplace_quad_p1", "stokes_momentum_hex_p1_vanilla",
                                 "laplace_hex_p4", "curl_curl_quad_p2"])
def test_nvrtc_compiles_for_sm100a(key):
    text, _, _ = fixture(key)
    plan = load_program(text)
    assert plan.config["cubin_bytes"] > 1000
    plan_fma = load_program(text, fma=True)
    assert plan_fma.config["cubin_bytes"] > 1000


def test_malformed_programs_raise_einval():
    with pytest.raises(NativeError) as e:
        load_program('{"name": "x"', jit=False)
    assert e.value.status == 1
    text, _, _ = fixture("action_mass_quad_p1")
    doc = json.loads(text)
    bad = json.loads(text)
    bad["body"].append(["frobnicate"])
    with pytest.raises(NativeError, match="unknown statement"):
        load_program(json.dumps(bad), jit=False)
    # unsupported math function (the reference raises UnsupportedFunction in emit_c)
    bad = json.loads(text)
    bad["body"].append(["assign", ["A", 0, []], ["call", "erf", ["lit", 1.0]]])
    with pytest.raises(NativeError, match="unsupported function"):
        load_program(json.dumps(bad), jit=False)
    # unknown buffer
    bad = json.loads(text)
    bad["body"].append(["assign", ["nope", 0, []], ["lit", 1.0]])
    with pytest.raises(NativeError, match="unknown buffer"):
        load_program(json.dumps(bad), jit=False)
    assert load_program(doc, jit=False).name == doc["name"]


def test_program_path_is_exported():
    lib = runtime.load_library()
    for s in ("sfk_program_create", "sfk_program_eval", "sfk_program_text"):
        assert hasattr(lib, s)


# ---------------------------------------------------------------------------
# GPU tier


@pytest.mark.gpu
@pytest.mark.parametrize("key", KEYS)
def test_gpu_bit_identical_to_reference(cuda, key):
    torch = cuda
    text, inputs, ref = fixture(key)
    plan = load_program(text)
    dev = {k: torch.from_numpy(v).cuda() for k, v in inputs.items()}
    out = evaluate_batched(plan, dev).cpu().numpy()
    if META[key]["transcendental"]:
        assert rel_err(out, ref) <= 1e-13
    else:
        assert np.array_equal(out, ref), rel_err(out, ref)


@pytest.mark.gpu
@pytest.mark.parametrize("key", ["action_laplace_hex_p3", "stokes_momentum_hex_p2",
                                 "laplace_hex_p4", "curl_curl_quad_p2_coffee",
                                 "stokes_momentum_hex_p1_vanilla"])
def test_gpu_fma_build_within_tolerance(cuda, key):
    torch = cuda
    text, inputs, ref = fixture(key)
    plan = load_program(text, fma=True)
    out = evaluate_batched(plan, {k: torch.from_numpy(v).cuda() for k, v in inputs.items()})
    assert rel_err(out.cpu().numpy(), ref) <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("p", [3, 4])
def test_gpu_program_matches_hand_kernel_on_lattice(cuda, p):
    """The same kernel two ways on 4096 lattice cells: the generated path from
    the reference's program and the hand-written C2 kernel."""
    torch = cuda
    text, _, _ = fixture("action_laplace_hex_p%d" % p)
    plan = load_program(text)
    inputs = workloads.c2_inputs(p, dims=(16, 16, 16))
    dev = {k: torch.from_numpy(v).cuda() for k, v in inputs.items()}
    a = evaluate_batched(plan, dev)
    b = evaluate_batched(compile_kernel("action_laplace", "hex", p), dev)
    assert rel_err(a.cpu().numpy(), b.cpu().numpy()) <= 1e-12


@pytest.mark.gpu
def test_gpu_run_kernel_semantics(cuda):
    torch = cuda
    text, inputs, ref = fixture("weighted_laplace_prism_p2")
    plan = load_program(text)
    # one cell, 1D inputs -> 1D output (interpreter.run_kernel calling convention)
    one = evaluate_batched(plan, {k: torch.from_numpy(v[3]).cuda() for k, v in inputs.items()})
    assert one.shape == (ref.shape[1],)
    assert np.array_equal(one.cpu().numpy(), ref[3])
    # numpy in -> numpy out
    out = evaluate_batched(plan, inputs)
    assert isinstance(out, np.ndarray) and np.array_equal(out, ref)
    # zero cells
    empty = {k: torch.zeros((0, v.shape[1]), dtype=torch.float64, device="cuda")
             for k, v in inputs.items()}
    assert evaluate_batched(plan, empty).shape == (0, ref.shape[1])
    # non-contiguous arguments
    nc = {k: torch.from_numpy(np.ascontiguousarray(v.T)).cuda().T for k, v in inputs.items()}
    assert np.array_equal(evaluate_batched(plan, nc).cpu().numpy(), ref)
    # launches are counted
    n0 = runtime.launch_count()
    evaluate_batched(plan, {k: torch.from_numpy(v).cuda() for k, v in inputs.items()})
    torch.cuda.synchronize()
    assert runtime.launch_count() == n0 + 1


@pytest.mark.gpu
def test_gpu_many_cells_partial_chunks(cuda):
    """Batches that are not multiples of the cells-per-CTA and exceed one wave."""
    torch = cuda
    text, inputs, ref = fixture("action_laplace_quad_p2")
    plan = load_program(text)
    reps = 1000
    big = {k: torch.from_numpy(np.tile(v, (reps, 1))[:-5].copy()).cuda() for k, v in inputs.items()}
    out = evaluate_batched(plan, big).cpu().numpy()
    assert np.array_equal(out, np.tile(ref, (reps, 1))[:-5])
