"""Simulation sharding plumbing.

The J simulations of Alg. 1 are independent samples, so a job of
J_total simulations is split over ranks by simulation: rank r builds simulations [j0, j1) with
im_build_sketches_shard and the library calls the collectives of its communicator at the points where
a greedy step needs all simulations (argmax values, the chosen vertex's score, sigma; include/im.h).
This module only computes the ranges and adapts torch.distributed to the communicator (or installs the
library's own NCCL communicator); all arithmetic is in the library's kernels.
"""
from __future__ import annotations

import numpy as np

IM_DTYPE_I32, IM_DTYPE_I64 = 0, 1
IM_OP_SUM, IM_OP_MAX = 0, 1
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


class TorchComm:
    """Host-side communicator for Library.im_set_comm over a torch.distributed process group (gloo for
    host-staged plumbing and tests; NCCL also works).  Each collective wraps the library's device buffer
    without a copy (CUDA array interface), runs the torch.distributed op and returns with the result in
    place.  Measured multi-GPU runs use the library's own NCCL communicator instead (nccl_init below)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.group = group
        self.rank = dist.get_rank(group)
        self.nranks = dist.get_world_size(group)
        self.host = dist.get_backend(group) == "gloo"

    def _t(self, ptr, count, dtype):
        import torch

        return torch.as_tensor(_DevArray(ptr, count, dtype), device="cuda")

    def _done(self):
        import torch

        torch.cuda.synchronize()

    def allreduce(self, ptr, count, dtype, op):
        import torch.distributed as dist

        t = self._t(ptr, count, dtype)
        h = t.cpu() if self.host else t
        dist.all_reduce(h, op=dist.ReduceOp.MAX if op == IM_OP_MAX else dist.ReduceOp.SUM, group=self.group)
        if self.host:
            t.copy_(h)
        self._done()

    def reduce_scatter(self, send, recv, recvcount, dtype):
        import torch.distributed as dist

        s = self._t(send, recvcount * self.nranks, dtype)
        r = self._t(recv, recvcount, dtype)
        if self.host:  # gloo has no reduce-scatter: sum everything, keep this rank's slice
            h = s.cpu()
            dist.all_reduce(h, group=self.group)
            r.copy_(h[self.rank * recvcount:(self.rank + 1) * recvcount])
        else:
            dist.reduce_scatter_tensor(r, s, group=self.group)
        self._done()

    def allgather(self, send, recv, sendcount, dtype):
        import torch
        import torch.distributed as dist

        s = self._t(send, sendcount, dtype)
        r = self._t(recv, sendcount * self.nranks, dtype)
        if self.host:
            parts = [torch.empty_like(s, device="cpu") for _ in range(self.nranks)]
            dist.all_gather(parts, s.cpu(), group=self.group)
            r.copy_(torch.cat(parts))
        else:
            dist.all_gather_into_tensor(r, s, group=self.group)
        self._done()


def nccl_init(lib, group=None):
    """Install the library's own NCCL communicator on every rank of a torch.distributed group: rank 0
    creates the ncclUniqueId, the 128 bytes are broadcast over the group (plumbing only)."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    obj = [lib.im_comm_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    lib.im_comm_nccl_init(obj[0], rank, world)
