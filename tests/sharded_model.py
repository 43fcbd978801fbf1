"""Host model of the simulation-sharded greedy step.

Test infrastructure: each rank holds simulations [j0, j1) (paper_2105_04023_b200.shard.shard_range)
of registers the oracle computed, and follows the library's exchange protocol (include/im.h,
im_build_sketches_shard): packed argmax values are reduce-scattered over vertex slices, the slice
argmaxes combined by a MAX all-reduce, the chosen vertex's score and the sigma count summed; every
decision is then taken from these.  Run over
gloo with world_size 2, the seeds / scores / step log must equal the unsharded oracle's.
"""
from __future__ import annotations

import math
import os

import numpy as np

import oracle
from paper_2105_04023_b200.shard import shard_range
from tests import brute

POOL_ONE = 1 << 24  # SHARD_POOL_ONE of csrc/im_internal.h


def pack_argmax(gain_local: np.ndarray, in_pool_local: np.ndarray) -> np.ndarray:
    return (gain_local.astype(np.int64) + in_pool_local.astype(np.int64) * POOL_ONE).astype(np.int32)


def unpack_argmax(summed: np.ndarray):
    s = summed.astype(np.int64)
    return s & (POOL_ONE - 1), (s >> 24) > 0


def sharded_select(n, off, tgt, pr, Jt, seed, K, eps_l, eps_g, rank, world, coll):
    """Alg. 1 on this rank's simulations with the library's exchange protocol
    (include/im.h): reduce-scatter of the packed per-vertex values, local argmax over this rank's vertex
    slice, MAX all-reduce of the 64-bit key (gain << 32 | ~v), SUM all-reduces of the chosen vertex's
    score and of the sigma count.  coll = (allreduce(arr, op), reduce_scatter(arr) -> slice)."""
    allreduce, reduce_scatter = coll
    j0, j1 = shard_range(Jt, rank, world)
    M = oracle.simulate(n, off, tgt, pr, Jt, seed)[0][:, j0:j1].astype(np.int64)
    MS = np.zeros(j1 - j0, np.int64)
    vis = np.zeros((n, j1 - j0), bool)
    S, steps, varsigma = [], [], 0.0
    Sl = -(-n // world)  # slice per rank, ceil(n / world)
    for k in range(K):
        gain = np.maximum(M - MS[None, :], 0).sum(axis=1)           # line 10, per rank
        inpool = ~vis.all(axis=1) if S else np.ones(n, bool)        # R14 pool, per rank
        packed = np.zeros(world * Sl, np.int32)
        packed[:n] = pack_argmax(gain, inpool)
        mine = reduce_scatter(packed)                                # exchange 1a: this rank's vertex slice
        g, pool = unpack_argmax(mine)
        v0 = rank * Sl
        key = 0
        for i in np.nonzero(pool)[0]:                                # local argmax, lowest id on ties
            v = v0 + int(i)
            if v < n:
                key = max(key, (int(g[i]) << 32) | (0xFFFFFFFF - v))
        key = int(allreduce(np.array([key], np.int64), "max")[0])   # exchange 1b
        if key:
            s = 0xFFFFFFFF - (key & 0xFFFFFFFF)
        else:
            s = int(next(v for v in range(n) if v not in S))
        score = allreduce(np.array([np.maximum(MS, M[s]).sum()], np.int64), "sum")[0]  # exchange 2
        S.append(s)
        full_reach = brute.reach_masks(n, off, tgt, pr, Jt, seed, S)
        vis = full_reach[:, j0:j1]
        cnt = allreduce(np.array([vis.sum()], np.int64), "sum")[0]  # exchange 3
        e = 2.0 ** (float(score) / Jt) / 0.77351                     # line 12
        sigma = float(cnt) / Jt
        delta = sigma - varsigma
        err_l = abs((e - delta) / delta) if delta != 0.0 else math.inf
        err_g = abs((e - delta) / sigma)
        rebuild = not (err_l < eps_l or err_g < eps_g)
        steps.append({"vertex": s, "score": int(score), "sigma_count": int(cnt), "rebuilt": int(rebuild)})
        if not rebuild:
            MS = np.maximum(MS, M[s])
        elif k < K - 1:
            varsigma = sigma
            MS[:] = 0
            M = oracle.simulate(n, off, tgt, pr, Jt, seed, blocked=full_reach)[0][:, j0:j1].astype(np.int64)
    return {"seeds": S, "steps": steps, "j0": j0, "j1": j1}


def gloo_worker(rank, world, port, case, out_q):
    """One rank of the world_size-`world` gloo run of sharded_select."""
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def allreduce(a, op):
        t = torch.from_numpy(a)
        dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
        return a

    def reduce_scatter(a):  # gloo: sum everything, keep this rank's slice
        t = torch.from_numpy(a.astype(np.int64))
        dist.all_reduce(t)
        Sl = len(a) // world
        return t.numpy()[rank * Sl:(rank + 1) * Sl].astype(np.int32)

    try:
        n, off, tgt, pr, Jt, seed, K, eps_l, eps_g = case
        r = sharded_select(n, off, tgt, pr, Jt, seed, K, eps_l, eps_g, rank, world, (allreduce, reduce_scatter))
        out_q.put((rank, r))
    finally:
        dist.destroy_process_group()
