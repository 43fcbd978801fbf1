"""Simulation sharding on CPU: shard ranges, and the sharded greedy protocol
over a real world_size-2 gloo process group against the unsharded oracle (-m "not gpu")."""
import math
import multiprocessing as mp
import socket

import numpy as np
import pytest

import oracle
from paper_2105_04023_b200.shard import shard_range
from tests import brute
from tests.sharded_model import gloo_worker, pack_argmax, unpack_argmax


def test_shard_range_partitions():
    for Jt in (32, 64, 96, 512, 1024, 2048, 4096):
        for world in range(1, 9):
            if Jt // 32 < world or Jt > 1024 * world:
                with pytest.raises(ValueError):
                    [shard_range(Jt, r, world) for r in range(world)]
                continue
            rs = [shard_range(Jt, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == Jt
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            sizes = [j1 - j0 for j0, j1 in rs]
            assert all(s % 32 == 0 and 32 <= s <= 1024 for s in sizes)
            assert max(sizes) - min(sizes) <= 32 and sizes == sorted(sizes, reverse=True)
    with pytest.raises(ValueError):
        shard_range(100, 0, 1)


def test_pack_roundtrip_sums():
    """Summed packed values decode to the summed gains and the OR of the pool flags (<= 127 ranks)."""
    rng = np.random.default_rng(0)
    parts = [(rng.integers(0, 32 * 1024, 50), rng.random(50) < 0.3) for _ in range(8)]
    tot = sum(pack_argmax(g, p).astype(np.int64) for g, p in parts).astype(np.int32)
    g, pool = unpack_argmax(tot)
    assert np.array_equal(g, sum(p[0] for p in parts))
    assert np.array_equal(pool, np.any([p[1] for p in parts], axis=0))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("Jt,eps", [(128, 0.05), (96, math.inf), (64, 0.0)])
def test_sharded_greedy_gloo_matches_oracle(Jt, eps):
    rng = np.random.default_rng(Jt)
    n = 40
    off, tgt, pr = brute.random_graph(rng, n, 120)
    K, seed = 6, 11
    case = (n, off, tgt, pr, Jt, seed, K, eps, eps)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=gloo_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    want = oracle.select_seeds(n, off, tgt, pr, Jt, seed, K, eps)
    assert res[0]["j0"] == 0 and res[0]["j1"] == res[1]["j0"] and res[1]["j1"] == Jt
    for r in (0, 1):
        assert res[r]["seeds"] == list(want["seeds"])
        for a, b in zip(res[r]["steps"], want["steps"]):
            assert (a["vertex"], a["score"], a["sigma_count"], a["rebuilt"]) == (b["vertex"], b["score"], b["sigma_count"], b["rebuilt"])
    if eps == 0.0:
        assert all(s["rebuilt"] for s in want["steps"])  # the rebuild path was exercised
