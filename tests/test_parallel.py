"""Multi-rank host logic on CPU (gloo, world_size 2) and the NCCL path on
one GPU.  The data path has no collective (cells are independent,
SPEC.md:580); only the scalar checksum all-reduce is exercised."""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import cpu
from paper_1711_02473_b200 import compile_kernel, workloads
from paper_1711_02473_b200.parallel import allreduce_sums, shard_range


def test_shard_range_partitions_exactly():
    for n in (0, 1, 7, 1000, 262144):
        for w in (1, 2, 3, 4, 8):
            ranges = [shard_range(n, r, w) for r in range(w)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            for (a, b), (c, d) in zip(ranges, ranges[1:]):
                assert b == c
            sizes = [b - a for a, b in ranges]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def test_lattice_slabs_tile_the_lattice():
    full = workloads.lattice_coords(4, 3, 2)
    parts = [workloads.lattice_coords(4, 3, 2, ix_range=(2 * r, 2 * r + 2)) for r in range(2)]
    assert np.array_equal(np.concatenate(parts), full)
    # C5 weak scaling: rank r of G owns its own 16-wide slab of a (16G,64,64) lattice
    a = workloads.c5_inputs(1, 2, (2, 3, 2))["coords"]
    b = workloads.lattice_coords(4, 3, 2, ix_range=(2, 4))
    assert np.array_equal(a, b)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, degree, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        inp = workloads.c5_inputs(rank, world, (2, 3, 2))
        plan = compile_kernel("laplace", "hex", degree)
        A = cpu.evaluate(plan, inp)          # stands in for the device kernel
        part = torch.tensor([float(np.sum(A * A)), float(np.sum(A))], dtype=torch.float64)
        allreduce_sums(part)
        q.put((rank, part.tolist(), inp["coords"].shape[0]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("degree", [1, 2])
def test_gloo_two_rank_checksum_matches_single_process(degree):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, degree, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sums = [r[1] for r in res]
    assert sums[0] == sums[1]                      # identical on every rank
    full = workloads.lattice_coords(2 * world, 3, 2)
    A = cpu.evaluate(compile_kernel("laplace", "hex", degree), {"coords": full})
    s2 = float(np.sum(A * A))
    assert abs(sums[0][0] - s2) <= 1e-12 * s2
    assert sum(r[2] for r in res) == full.shape[0]


@pytest.mark.gpu
def test_nccl_checksum_single_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    from paper_1711_02473_b200.parallel import sharded_matrix_checksum

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", str(_free_port()))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        norm, total, nloc = sharded_matrix_checksum(2, dims_per_rank=(2, 4, 4))
    finally:
        dist.destroy_process_group()
    A = cpu.evaluate(compile_kernel("laplace", "hex", 2),
                     {"coords": workloads.c5_inputs(0, 1, (2, 4, 4))["coords"]})
    assert nloc == 32
    assert abs(norm - math.sqrt(np.sum(A * A))) <= 1e-12 * norm


def _gpu_worker(rank, world, port, degree, q):
    """One rank of a 2-process run on ONE GPU: real kernels (sfk_eval through
    sharded_matrix_checksum), gloo all-reduce of the checksum partials.  The
    ranks never wait on each other's kernels (only the host all-reduce)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1711_02473_b200 import parallel

        norm, total, nloc = parallel.sharded_matrix_checksum(degree, dims_per_rank=(2, 3, 2))
        q.put((rank, norm, total, nloc))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("degree", [1, 3])
def test_two_ranks_one_gpu_real_kernels_checksum(degree):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, world, port, degree, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][1:3] == res[1][1:3]              # identical on every rank
    full = workloads.lattice_coords(2 * world, 3, 2)
    A = cpu.evaluate(compile_kernel("laplace", "hex", degree), {"coords": full})
    s2 = float(np.sum(A * A))
    assert abs(res[0][1] - math.sqrt(s2)) <= 1e-12 * math.sqrt(s2)
    assert sum(r[3] for r in res) == full.shape[0]


@pytest.mark.gpu
def test_bench_two_ranks_shared_device():
    """bench.py --gpus 2 relaunches itself under torch.distributed.run (one
    process per rank) and reports the aggregate of both ranks.  On this 1-GPU
    box both ranks share cuda:0 over gloo (--shared-device, test only)."""
    import json
    import subprocess
    import sys

    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2",
                          "--backend", "gloo", "--shared-device", "--steps", "2", "--warmup", "1",
                          "--degrees", "1-3", "--lattice", "8,8,8", "--c5-lattice", "2,4,4",
                          "--no-cpu"], capture_output=True, text=True, timeout=900, cwd=root)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [json.loads(l) for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]
    d = lines[0]
    assert d["n_gpus"] == 2 and d["config"]["cells_total"] == 2 * 512
    assert d["e2e"]["matches_device_path"] and d["gpu_launches"] > 0
    c5 = d["c5"]["per_degree"]
    assert [r["p"] for r in c5] == [1, 2, 3, 4]
    # checksum of the 2-rank lattice (4, 4, 4) equals the single-process one
    full = workloads.lattice_coords(4, 4, 4)
    for r in c5[:2]:
        A = cpu.evaluate(compile_kernel("laplace", "hex", r["p"]), {"coords": full})
        ref = math.sqrt(float(np.sum(A * A)))
        assert abs(r["frobenius"] - ref) <= 1e-12 * ref
