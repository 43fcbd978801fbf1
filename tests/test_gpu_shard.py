"""Simulation sharding on one GPU: two library contexts (two copies of the
.so, one thread each) hold the two halves of the simulations and exchange through an in-process
communicator (the im_comm protocol of include/im.h: reduce-scatter, all-reduce sum / max, all-gather).  Every rank's seeds, scores, step log and estimates must equal the unsharded
context's, and its registers / reach bits must equal the unsharded columns [j0, j1).

The ranks only wait for each other on the host (inside the collectives, with the library's stream
drained), never inside a kernel, so running them on one GPU is safe."""
import os
import shutil
import tempfile
import threading

import numpy as np
import pytest

import gen
import paper_2105_04023_b200 as im
from paper_2105_04023_b200.shard import _DevArray, shard_range
from tests import brute

pytestmark = pytest.mark.gpu

_libs = []


def shard_libs(world):
    while len(_libs) < world:
        d = tempfile.mkdtemp(prefix="im_shard_")
        p = os.path.join(d, f"libim_b200_rank{len(_libs)}.so")
        shutil.copy(im.LIB_PATH, p)
        _libs.append(im.Library(p))
    return _libs[:world]


class ThreadComm:
    """The communicator protocol (include/im.h im_comm) over `world` threads of one process, host-staged:
    device -> host, combine, host -> device."""

    def __init__(self, world):
        import torch

        self.torch = torch
        self.world = world
        self.bar = threading.Barrier(world, timeout=300)
        self.parts = [None] * world
        self.calls = 0

    def _gather(self, rank, arr):
        self.parts[rank] = arr
        self.bar.wait()
        allp = list(self.parts)
        self.bar.wait()
        return allp

    def comm(self, rank):
        torch, tc = self.torch, self

        class C:
            nranks = tc.world

            def __init__(self):
                self.rank = rank

            def allreduce(self, ptr, count, dtype, op):
                t = torch.as_tensor(_DevArray(ptr, count, dtype), device="cuda")
                allp = tc._gather(rank, t.cpu().numpy().astype(np.int64))
                tot = np.max(allp, axis=0) if op == im.IM_OP_MAX else np.sum(allp, axis=0)
                t.copy_(torch.from_numpy(tot.astype(t.cpu().numpy().dtype)))
                torch.cuda.synchronize()
                if rank == 0:
                    tc.calls += 1

            def reduce_scatter(self, send, recv, recvcount, dtype):
                s = torch.as_tensor(_DevArray(send, recvcount * tc.world, dtype), device="cuda")
                r = torch.as_tensor(_DevArray(recv, recvcount, dtype), device="cuda")
                allp = tc._gather(rank, s.cpu().numpy().astype(np.int64))
                tot = np.sum(allp, axis=0)[rank * recvcount:(rank + 1) * recvcount]
                r.copy_(torch.from_numpy(tot.astype(r.cpu().numpy().dtype)))
                torch.cuda.synchronize()

            def allgather(self, send, recv, sendcount, dtype):
                s = torch.as_tensor(_DevArray(send, sendcount, dtype), device="cuda")
                r = torch.as_tensor(_DevArray(recv, sendcount * tc.world, dtype), device="cuda")
                allp = tc._gather(rank, s.cpu().numpy())
                r.copy_(torch.from_numpy(np.concatenate(allp)))
                torch.cuda.synchronize()

        return C()


def run_sharded(world, n, off, tgt, pr, Jt, seed, K, eps, want_est=True):
    libs = shard_libs(world)
    tcomm = ThreadComm(world)
    out = [None] * world
    err = []

    def rank_main(r):
        try:
            L = libs[r]
            j0, j1 = shard_range(Jt, r, world)
            L.im_set_comm(tcomm.comm(r))  # before the build: it sizes the exchange buffers
            L.im_load_csr(n, off, tgt, pr)
            L.im_build_sketches_shard(Jt, seed, j0, j1)
            est = L.im_estimate(n) if want_est else None
            s, sc = L.im_select_seeds(K, eps)
            out[r] = {"j0": j0, "j1": j1, "seeds": s, "scores": sc, "log": L.im_get_step_log(K), "est": est,
                      "M": L.im_get_registers(n, j1 - j0), "reach": L.im_get_reach(n, j1 - j0),
                      "stats": L.im_get_stats()}
        except Exception as e:  # surfaced below
            err.append((r, e))
            tcomm.bar.abort()

    ts = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not err, err
    return out, tcomm.calls


def unsharded(n, off, tgt, pr, J, seed, K, eps):
    im.im_load_csr(n, off, tgt, pr)
    im.im_build_sketches(J, seed)
    est = im.im_estimate(n)
    M0 = im.im_get_registers(n, J)
    s, sc = im.im_select_seeds(K, eps)
    return {"seeds": s, "scores": sc, "log": im.im_get_step_log(K), "est": est, "M0": M0, "reach": im.im_get_reach(n, J)}


def check_equal(out, ref, n, J, check_regs=True):
    vis = im.reach_bits_to_bool(ref["reach"], J)
    for o in out:
        assert list(o["seeds"]) == list(ref["seeds"])
        assert list(o["scores"]) == list(ref["scores"])
        assert o["log"] == ref["log"]
        if o["est"] is not None:
            assert np.array_equal(o["est"], ref["est"])
        j0, j1 = o["j0"], o["j1"]
        assert o["stats"]["J_total"] == J and o["stats"]["j0"] == j0 and o["stats"]["J"] == j1 - j0
        assert np.array_equal(im.reach_bits_to_bool(o["reach"], j1 - j0), vis[:, j0:j1])


@pytest.mark.parametrize("J,world,eps", [(128, 2, 0.05), (96, 2, 0.0), (256, 3, float("inf"))])
def test_sharded_small_matches_unsharded(J, world, eps):
    rng = np.random.default_rng(J + world)
    n = 300
    off, tgt, pr = brute.random_graph(rng, n, 1500)
    K, seed = 12, 5
    ref = unsharded(n, off, tgt, pr, J, seed, K, eps)
    out, calls = run_sharded(world, n, off, tgt, pr, J, seed, K, eps)
    assert calls >= 2 * K
    check_equal(out, ref, n, J)
    # first-build registers of each shard == the unsharded columns (rebuilds may have replaced
    # the final ones, so compare a fresh shard build)
    libs = shard_libs(world)
    for r, o in enumerate(out):
        L = libs[r]
        L.im_build_sketches_shard(J, seed, o["j0"], o["j1"])
        assert np.array_equal(L.im_get_registers(n, o["j1"] - o["j0"]), ref["M0"][:, o["j0"]:o["j1"]])


def test_shard_validation_and_state():
    n, off, tgt, pr = 10, np.arange(11, dtype=np.int32), np.arange(1, 11, dtype=np.int32) % 10, np.full(10, 0.5, np.float32)
    L = shard_libs(1)[0]
    L.im_set_comm(None)
    L.im_load_csr(n, off, tgt, pr)
    for args in [(64, 1, 0, 16), (64, 1, 32, 32), (64, 1, 32, 96), (100, 1, 0, 32), (4096, 1, 0, 2048)]:
        with pytest.raises(im.IMError) as e:
            L.im_build_sketches_shard(*args)
        assert e.value.code == im.IM_EINVAL
    L.im_build_sketches_shard(64, 1, 32, 64)
    with pytest.raises(im.IMError) as e:  # sharded sketches without a communicator
        L.im_select_seeds(2, 0.1)
    assert e.value.code == im.IM_ESTATE

    class Bad:
        rank, nranks = 0, 2

        def allreduce(self, *a):
            raise RuntimeError("peer gone")

        reduce_scatter = allgather = allreduce

    L.im_set_comm(Bad())
    with pytest.raises(im.IMError) as e:  # communicator changed after the build
        L.im_estimate(n)
    assert e.value.code == im.IM_ESTATE
    L.im_build_sketches_shard(64, 1, 32, 64)
    with pytest.raises(im.IMError) as e:
        L.im_estimate(n)
    assert e.value.code == im.IM_ECOMM

    class BadRank(Bad):
        rank, nranks = 3, 2

    with pytest.raises(im.IMError) as e:
        L.im_set_comm(BadRank())
    assert e.value.code == im.IM_EINVAL
    L.im_set_comm(None)
    L.im_build_sketches_shard(64, 1, 0, 64)  # whole range: an ordinary context again
    s, _ = L.im_select_seeds(2, 0.1)
    assert len(s) == 2


def test_sharded_c3_matches_unsharded():
    """C3 (4M vertices, J = 256) split over 2 ranks: identical K = 50 selection."""
    cfg = gen.CONFIGS["c3"]
    from tests.test_gpu_configs import cached_graph

    n, off, tgt = cached_graph(cfg.graph)
    pr = np.full(len(tgt), cfg.p, np.float32)
    im.im_load_csr(n, off, tgt, pr)
    im.im_build_sketches(cfg.J, cfg.salt_seed)
    s, sc = im.im_select_seeds(cfg.K, cfg.t)
    log = im.im_get_step_log(cfg.K)
    out, _ = run_sharded(2, n, off, tgt, pr, cfg.J, cfg.salt_seed, cfg.K, cfg.t, want_est=False)
    for o in out:
        assert list(o["seeds"]) == list(s) and list(o["scores"]) == list(sc) and o["log"] == log
