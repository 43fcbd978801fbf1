"""Simulation sharding across PROCESSES (include/im.h im_comm): world_size 2 and 3
gloo groups, one process and one libim_b200.so context per rank (tests/mp_shard_worker.py), the
communicator's reduce-scatter / all-reduce / all-gather exchanges.  Every rank's seeds, scores, step
log and estimates must equal the unsharded oracle's (Alg. 1), and its reach bits
the oracle's R_G(S) columns [j0, j1)."""
import math
import multiprocessing as mp
import socket

import numpy as np
import pytest

import gen
import oracle
import paper_2105_04023_b200 as im
from tests import brute

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def run_ranks(world, case):
    from tests.mp_shard_worker import rank_main

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=rank_main, args=(r, world, port, case, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=600) for _ in ps)
    for p in ps:
        p.join(120)
    for r in range(world):
        assert "error" not in res[r], res[r]
    assert all(p.exitcode == 0 for p in ps)
    return res


def cases():
    c1 = gen.CONFIGS["c1"]
    n, off, tgt, pr = gen.workload(c1)
    out = [pytest.param(2, (n, off, tgt, pr, c1.J, c1.salt_seed, c1.K, c1.t, c1.t), id="c1-world2")]
    rng = np.random.default_rng(77)
    off2, tgt2, pr2 = brute.random_graph(rng, 600, 4000)
    out.append(pytest.param(3, (600, off2, tgt2, pr2, 160, 3, 12, 0.3, 0.01), id="random-world3-paper-policy"))
    out.append(pytest.param(2, (600, off2, tgt2, pr2, 128, 4, 8, 0.0, 0.0), id="random-world2-always-rebuild"))
    return out


@pytest.mark.parametrize("world,case", cases())
def test_multiprocess_shards_match_oracle(world, case):
    n, off, tgt, pr, Jt, seed, K, eps_l, eps_g = case
    res = run_ranks(world, case)
    want = oracle.select_seeds(n, off, tgt, pr, Jt, seed, K, eps_l, eps_g, want_vis=True)
    M, _ = oracle.simulate(n, off, tgt, pr, Jt, seed)
    est = oracle.estimate(M)
    j_prev = 0
    for r in range(world):
        o = res[r]
        assert o["j0"] == j_prev and o["stats"]["J_total"] == Jt
        j_prev = o["j1"]
        assert o["seeds"] == list(want["seeds"])
        assert o["scores"] == list(want["scores"])
        for a, b in zip(o["log"], want["steps"]):
            assert (a["vertex"], a["score"], a["sigma_count"], a["rebuilt"], a["executed"]) == \
                (b["vertex"], b["score"], b["sigma_count"], b["rebuilt"], b["executed"])
        assert np.all(np.abs(o["est"] - est) <= 1e-6 * est)
        vis = im.reach_bits_to_bool(o["reach"], o["j1"] - o["j0"])
        assert np.array_equal(vis, want["vis"][:, o["j0"]:o["j1"]].astype(bool))
    assert j_prev == Jt
    if eps_l == 0.0:
        assert all(s["rebuilt"] for s in want["steps"])
