"""Multi-GPU: cell-range sharding and scalar all-reduces.

Cells are independent and the reference kernel is a pure per-cell function
(SPEC.md:580), so the hot path has no exchange step: rank r owns the
contiguous cell range ``shard_range(C, r, G)`` (or, for lattice workloads,
the slab ``ix in [nx*r, nx*(r+1))``) and runs ``evaluate_batched`` on it with
no collective.  The only communication is an all-reduce of a handful of
fp64 scalars after the kernels — the Frobenius checksum of BASELINE config
C5 and functionals such as sum(A) — through ``torch.distributed``
(NCCL over NVLink/NVSwitch on GPUs, gloo in the CPU tests).  The payload is
~16 bytes, so there is nothing to fuse or overlap: latency only.
"""

from __future__ import annotations

import math

__all__ = ["shard_range", "rank_world", "allreduce_sums", "frobenius_checksum",
           "sharded_matrix_checksum"]


def shard_range(ncells, rank, world):
    """Contiguous, balanced [lo, hi) of rank ``rank`` out of ``world``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world %d/%d" % (rank, world))
    base, extra = divmod(int(ncells), world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def rank_world():
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def allreduce_sums(partials, group=None):
    """All-reduce (SUM) a small float64 tensor of per-rank partial sums.

    ``partials`` lives on the device matching the process group's backend
    (CUDA for NCCL, CPU for gloo).  Returns the reduced tensor (in place).
    Ranks contribute in a fixed order inside the collective, so the result
    is identical on every rank.
    """
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        if partials.is_cuda and dist.get_backend(group) == "gloo":
            host = partials.cpu()                # gloo reduces host tensors
            dist.all_reduce(host, op=dist.ReduceOp.SUM, group=group)
            partials.copy_(host)
        else:
            dist.all_reduce(partials, op=dist.ReduceOp.SUM, group=group)
    return partials


def frobenius_checksum(A, group=None, workspace=None):
    """Global ||A||_F and sum(A) over all ranks' local arrays.

    The local partials (sum A^2, sum A) come from the device reduction
    ``sfk_sum_squares`` (deterministic order); the cross-rank sum is one
    NCCL all-reduce of 2 doubles.
    """
    from .runtime import sum_squares

    part = sum_squares(A.reshape(-1), workspace=workspace).clone()
    allreduce_sums(part, group)
    s2, s1 = part.tolist()
    return math.sqrt(s2), s1


def sharded_matrix_checksum(degree, rank=None, world=None, dims_per_rank=(16, 64, 64),
                            device=None):
    """BASELINE config C5 end to end: rank r assembles the local Laplace
    matrices of its (16, 64, 64) slab of a (16*G, 64, 64) lattice and the
    Frobenius checksum is all-reduced.  Returns (norm, sum, local_cells)."""
    import torch

    from . import workloads
    from .plan import compile_kernel
    from .runtime import evaluate_batched

    if rank is None or world is None:
        rank, world = rank_world()
    inp = workloads.c5_inputs(rank, world, dims_per_rank)
    dev = device or torch.device("cuda", torch.cuda.current_device())
    coords = torch.from_numpy(inp["coords"]).to(dev)
    plan = compile_kernel("laplace", "hex", degree)
    A = evaluate_batched(plan, {"coords": coords})
    norm, total = frobenius_checksum(A)
    return norm, total, coords.shape[0]
