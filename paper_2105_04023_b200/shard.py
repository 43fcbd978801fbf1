"""Simulation sharding plumbing.

The J simulations of Alg. 1 are independent samples, so a job of
J_total simulations is split over ranks by simulation: rank r builds simulations [j0, j1) with
im_build_sketches_shard and the library calls the allreduce hook at the three points where
a greedy step needs all simulations (argmax values, the chosen vertex's score, sigma).  This
module only computes the ranges and adapts torch.distributed to the hook; all arithmetic is in
the library's kernels.
"""
from __future__ import annotations

import numpy as np

IM_DTYPE_I32, IM_DTYPE_I64 = 0, 1
_NP = {IM_DTYPE_I32: np.int32, IM_DTYPE_I64: np.int64}
_TYPESTR = {IM_DTYPE_I32: "<i4", IM_DTYPE_I64: "<i8"}


def shard_range(J_total: int, rank: int, world: int) -> tuple[int, int]:
    """[j0, j1) of rank `rank`: whole 32-simulation words, as even as possible (earlier ranks
    never get fewer).  Raises if some rank would get no word or more than 1024 simulations."""
    if J_total % 32 or J_total < 32:
        raise ValueError(f"J_total must be a positive multiple of 32 (got {J_total})")
    if world >= 256:  # the packed argmax value counts in-pool ranks in 8 bits (gain + count << 24)
        raise ValueError(f"world size {world} >= 256 is not supported by the packed argmax exchange")
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} not in [0, {world})")
    words = J_total // 32
    if words < world:
        raise ValueError(f"{J_total} simulations cannot be split over {world} ranks (32 per rank minimum)")
    base, extra = divmod(words, world)
    w0 = rank * base + min(rank, extra)
    w1 = w0 + base + (1 if rank < extra else 0)
    if (w1 - w0) * 32 > 1024:
        raise ValueError(f"rank {rank} would hold {(w1 - w0) * 32} > 1024 simulations; use more ranks")
    return 32 * w0, 32 * w1


class _DevArray:
    """Zero-copy view of library device memory for torch.as_tensor (CUDA array interface v3)."""

    def __init__(self, ptr: int, count: int, dtype: int):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": _TYPESTR[dtype], "data": (ptr, False),
                                         "version": 3, "strides": None, "stream": None}


def torch_allreduce_hook(group=None):
    """Hook for Library.im_set_allreduce over a torch.distributed process group (NCCL): wraps the
    library's buffer without a copy, all_reduce(SUM) on torch's current stream, waits for it."""
    import torch
    import torch.distributed as dist

    def hook(ptr: int, count: int, dtype: int) -> None:
        t = torch.as_tensor(_DevArray(ptr, count, dtype), device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        torch.cuda.current_stream().synchronize()

    return hook


def host_allreduce(buf: np.ndarray, group=None) -> np.ndarray:
    """The same SUM for a host array through torch.distributed (gloo); used by the CPU tests of the
    sharded protocol.  In place; returns buf."""
    import torch
    import torch.distributed as dist

    t = torch.from_numpy(buf)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return buf
