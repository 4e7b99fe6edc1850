"""bench.py's reference arm (CPU, no GPU needed): one JSON line with the
driver's keys; the CPU baseline reports both SURVEY §8(d) builds."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ref_available():
    sys.path.insert(0, ROOT)
    from oracle import refc
    from paper_1711_02473_b200 import compile_kernel
    return all(refc.available(compile_kernel("action_laplace", "hex", p)) for p in (1, 2))


def test_reference_arm_json_line():
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "1", "--degrees", "1-2",
                          "--cpu-cells", "512"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["unit"] == "GDoF/s" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    cb = d["cpu_baseline"]
    assert cb["value"] == d["value"] and cb["cores"] >= 1 and cb["kind"] in ("reference", "port")
    if cb["kind"] == "reference":
        assert set(cb["by_build"]) <= {"parity", "fast"} and cb["build"] in cb["by_build"]


@pytest.mark.skipif(not os.path.isdir(os.path.join(ROOT, "oracle", "_ref")), reason="no oracle/_ref")
def test_cpu_baseline_leg_reports_both_builds_and_single_thread():
    if not _ref_available():
        pytest.skip("reference C not built")
    sys.path.insert(0, ROOT)
    import bench
    from paper_1711_02473_b200 import workloads
    degs = [1, 2]
    coords = workloads.lattice_coords(8, 8, 8)
    hu = {p: workloads.uniform_dofs(coords.shape[0], (p + 1) ** 3) for p in degs}
    dev_out = {p: bench_ref(p, coords, hu[p]) for p in degs}
    cb, parity = bench.cpu_baseline_leg(degs, coords, hu, 256, dev_out)
    assert cb["kind"] == "reference" and cb["value"] > 0 and cb["cpu_model"]
    assert cb["single_thread"]["value"] > 0
    assert cb["compiled_on_this_host"]
    # the parity check itself: the oracle port vs the reference C, first 256 cells
    assert set(parity) == set(degs) and max(parity.values()) < 1e-12


def bench_ref(p, coords, u):
    from oracle import cpu
    from paper_1711_02473_b200 import compile_kernel
    return cpu.evaluate(compile_kernel("action_laplace", "hex", p), {"coords": coords, "w0": u})


def test_parity_err_metric():
    import numpy as np
    sys.path.insert(0, ROOT)
    import bench
    ref = np.array([[1.0, -2.0, 0.5], [0.0, 0.0, 1e-3]])
    assert bench.parity_err(ref, ref) == 0.0
    x = ref.copy()
    x[0, 1] += 2e-12       # 1e-12 relative to the cell's max |y| = 2
    assert abs(bench.parity_err(x, ref) - 1e-12) < 1e-15
    x = ref.copy()
    x[1, 0] = np.nan       # NaN where the reference is finite
    assert bench.parity_err(x, ref) == float("inf")


def test_gpus_flag_must_match_world_size():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4",
                          "--impl", "reference"], capture_output=True, text=True, env=env,
                         timeout=300, cwd=ROOT)
    assert res.returncode != 0 and "WORLD_SIZE" in res.stderr
