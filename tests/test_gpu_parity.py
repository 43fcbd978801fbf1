"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle on the same seeded inputs.

Bar (BASELINE.json north_star): registers, reach masks and seed sets bit-exact; estimates
within 1e-6 relative (double accumulation); seed picks whose competing estimates differ by
< 1e-6 relative are reported, not failed (none can occur here: the argmax is over exact
integer sums with a lowest-id tie break on both sides).
"""
import math

import numpy as np
import pytest

import oracle
import paper_2105_04023_b200 as im
from tests import brute

pytestmark = pytest.mark.gpu

EST_RTOL = 1e-6


def run_build(n, off, tgt, pr, J, seed):
    im.im_load_csr(n, off, tgt, pr)
    im.im_build_sketches(J, seed)
    return im.im_get_registers(n, J)


def reach_bool(n, J):
    return im.reach_bits_to_bool(im.im_get_reach(n, J), J)


# ------------------------------------------------------------------ validation / edge cases
def test_validation_errors():
    bad = [
        (3, [0, 1, 2, 2], [1, 3], [0.5, 0.5]),       # target out of range
        (3, [0, 2, 1, 2], [1, 2], [0.5, 0.5]),       # decreasing offsets
        (3, [0, 1, 2, 2], [1, 2], [0.5, float("nan")]),
        (3, [0, 1, 2, 2], [1, 2], [0.5, 1.5]),
        (3, [0, 1, 2, 2], [1, 2], [-0.1, 0.5]),
    ]
    for n, o, t, p in bad:
        with pytest.raises(im.IMError) as e:
            im.im_load_csr(n, o, t, p)
        assert e.value.code == im.IM_EINVAL
    im.im_load_csr(3, [0, 1, 2, 2], [1, 2], [0.5, 0.5])
    for J in (0, 16, 48, 2048):
        with pytest.raises(im.IMError) as e:
            im.im_build_sketches(J, 1)
        assert e.value.code == im.IM_EINVAL
    with pytest.raises(im.IMError) as e:
        im.im_select_seeds(1, 0.05)
    assert e.value.code == im.IM_ESTATE
    im.im_build_sketches(32, 1)
    for K, t in ((4, 0.05), (-1, 0.05), (1, float("nan")), (1, -1.0)):
        with pytest.raises(im.IMError) as e:
            im.im_select_seeds(K, t)
        assert e.value.code == im.IM_EINVAL
    s, sc = im.im_select_seeds(0, 0.05)
    assert len(s) == 0


def test_degenerate_graphs():
    """n = 1, no edges, all-zero / all-one probabilities, self loops and duplicates only."""
    cases = [
        (1, [0, 0], [], []),
        (5, [0] * 6, [], []),
        (2, [0, 1, 1], [1], [0.5]),                   # a single edge (per-edge threshold path)
        (3, [0, 0, 1, 1], [0], [1.0]),
        (4, [0, 2, 3, 3, 4], [1, 1, 2, 0], [0.0, 0.0, 0.0, 0.0]),
        (4, [0, 2, 3, 3, 4], [1, 1, 2, 0], [1.0, 1.0, 1.0, 1.0]),
        (3, [0, 2, 4, 4], [0, 0, 1, 1], [1.0, 0.7, 1.0, 0.2]),
    ]
    for n, o, t, p in cases:
        for J in (32, 64):
            o_, t_, p_ = np.array(o, np.int32), np.array(t, np.int32), np.array(p, np.float32)
            M = run_build(n, o_, t_, p_, J, 5)
            Mo, _ = oracle.simulate(n, o_, t_, p_, J, 5)
            assert np.array_equal(M, Mo)
            K = min(n, 3)
            for thr in (0.0, math.inf):
                s, sc = im.im_select_seeds(K, thr)
                r = oracle.select_seeds(n, o_, t_, p_, J, 5, K, thr)
                assert list(s) == list(r["seeds"]) and list(sc) == list(r["scores"])


# ------------------------------------------------------------------ registers (Alg. 2)
@pytest.mark.parametrize("J", [32, 64, 96, 128, 256, 512, 1024])
def test_registers_random_graphs(J):
    rng = np.random.default_rng(100 + J)
    for g in range(7):
        n = int(rng.integers(2, 3000 if J <= 256 else 800))
        m = int(rng.integers(0, 6 * n))
        # 0.001: more than 2^8 hash buckets per row, the radix-sort edge prep (im_prep.cu)
        p = [None, 0.005, 0.05, 0.3, 1.0, 0.01, 0.001][g]
        off, tgt, pr = brute.random_graph(rng, n, m, p)
        seed = int(rng.integers(0, 2**63))
        M = run_build(n, off, tgt, pr, J, seed)
        Mo, _ = oracle.simulate(n, off, tgt, pr, J, seed)
        assert np.array_equal(M, Mo), (J, g, n, m, p)


def test_registers_tiny_vs_bruteforce():
    rng = np.random.default_rng(7)
    for g in range(25):
        n = int(rng.integers(2, 60))
        off, tgt, pr = brute.random_graph(rng, n, int(rng.integers(0, 4 * n)), None)
        M = run_build(n, off, tgt, pr, 32, g)
        assert np.array_equal(M, brute.registers(n, off, tgt, pr, 32, g))


def test_hub_and_wide_windows():
    """A 20k-out/in-degree hub (multi-segment work items) and w = 1 / WC edges (dense windows)."""
    rng = np.random.default_rng(3)
    n = 25000
    src = np.concatenate([np.zeros(20000, np.int64), rng.integers(0, n, 40000), rng.integers(0, n, 20000)])
    dst = np.concatenate([rng.integers(1, n, 20000), rng.integers(0, n, 40000), np.zeros(20000, np.int64)])
    order = np.lexsort((dst, src))
    src, dst = src[order], dst[order]
    off = np.zeros(n + 1, np.int64)
    np.add.at(off, src + 1, 1)
    off = np.cumsum(off).astype(np.int32)
    tgt = dst.astype(np.int32)
    indeg = np.bincount(tgt, minlength=n)
    for pr in (np.full(len(tgt), 0.02, np.float32), np.full(len(tgt), 0.001, np.float32), (1.0 / indeg[tgt]).astype(np.float32)):
        for J in (64, 512):
            M = run_build(n, off, tgt, pr, J, 11)
            Mo, _ = oracle.simulate(n, off, tgt, pr, J, 11)
            assert np.array_equal(M, Mo)


# ------------------------------------------------------------------ estimate (Eq. 2)
def test_estimate_parity():
    rng = np.random.default_rng(5)
    for J in (32, 256, 1024):
        n = 3000
        off, tgt, pr = brute.random_graph(rng, n, 4 * n, 0.1)
        M = run_build(n, off, tgt, pr, J, 9)
        e = im.im_estimate(n)
        eo = oracle.estimate(M)
        assert np.all(np.abs(e - eo) <= EST_RTOL * eo)
        assert np.max(np.abs(e - eo) / eo) < 1e-14  # exact integer sums + one exp2


# ------------------------------------------------------------------ greedy (Alg. 1)
def test_constant_w_entry_point_vs_oracle():
    """im_load_csr_const (one scalar w, the paper's constant-probability settings PAPER.md:457-462) against the
    oracle run on the explicit array: registers, seeds, scores and reach; degenerate sizes and a bad w."""
    rng = np.random.default_rng(77)
    for g, (w, J) in enumerate([(0.005, 64), (0.01, 128), (0.1, 256), (1.0, 32), (0.0, 32), (0.3, 96)]):
        n = int(rng.integers(2, 2500))
        m = int(rng.integers(2, 6 * n))
        off, tgt, pr = brute.random_graph(rng, n, m, w)
        seed = int(rng.integers(0, 2**63))
        im.im_load_csr_const(n, off, tgt, w)
        im.im_build_sketches(J, seed)
        st = im.im_get_stats()
        assert st["const_threshold"] == 1
        Mo, _ = oracle.simulate(n, off, tgt, pr, J, seed)
        assert np.array_equal(im.im_get_registers(n, J), Mo), (g, n, m, w)
        K = min(n, 8)
        s, sc = im.im_select_seeds(K, 0.05)
        r = oracle.select_seeds(n, off, tgt, pr, J, seed, K, 0.05, want_vis=True)
        assert list(s) == list(r["seeds"]) and list(sc) == list(r["scores"])
        assert np.array_equal(reach_bool(n, J), r["vis"].astype(bool))
    # no edge / one edge (the array path inside), device pointers
    for off, tgt in (([0, 0, 0], []), ([0, 1, 1], [1])):
        im.im_load_csr_const(2, off, tgt, 0.5)
        im.im_build_sketches(32, 3)
        Mo, _ = oracle.simulate(2, np.array(off, np.int32), np.array(tgt, np.int32), np.full(len(tgt), 0.5, np.float32), 32, 3)
        assert np.array_equal(im.im_get_registers(2, 32), Mo)
    import torch
    n, m = 500, 3000
    off, tgt, pr = brute.random_graph(rng, n, m, 0.05)
    d_off, d_tgt = torch.from_numpy(off).cuda(), torch.from_numpy(tgt).cuda()
    torch.cuda.synchronize()
    im.im_load_csr_const_device(n, len(tgt), d_off, d_tgt, 0.05)
    im.im_build_sketches(64, 5)
    Mo, _ = oracle.simulate(n, off, tgt, pr, 64, 5)
    assert np.array_equal(im.im_get_registers(n, 64), Mo)
    for w in (float("nan"), 1.5, -0.1):
        with pytest.raises(im.IMError) as e:
            im.im_load_csr_const(n, off, tgt, w)
        assert e.value.code == im.IM_EINVAL


def compare_select(n, off, tgt, pr, J, seed, K, t):
    im.im_load_csr(n, off, tgt, pr)
    im.im_build_sketches(J, seed)
    s, sc = im.im_select_seeds(K, t)
    log = im.im_get_step_log(K)
    r = oracle.select_seeds(n, off, tgt, pr, J, seed, K, t, want_vis=True)
    assert list(s) == list(r["seeds"]), (list(s), list(r["seeds"]))
    assert list(sc) == list(r["scores"])
    for a, b in zip(log, r["steps"]):
        assert a["vertex"] == b["vertex"] and a["score"] == b["score"] and a["sigma_count"] == b["sigma_count"]
        assert a["rebuilt"] == b["rebuilt"] and a["executed"] == b["executed"]
        for f in ("e", "sigma", "delta", "err_l", "err_g"):
            x, y = a[f], b[f]
            assert (x == y) or (math.isinf(x) and math.isinf(y)) or abs(x - y) <= 1e-12 * max(abs(x), abs(y)), (f, x, y)
    assert np.array_equal(reach_bool(n, J), r["vis"].astype(bool))
    return r


@pytest.mark.parametrize("t", [0.0, 0.05, 0.3, math.inf])
def test_select_parity_random(t):
    rng = np.random.default_rng(int(1000 * (t if t != math.inf else 9)))
    for g in range(5):
        n = int(rng.integers(50, 1500))
        off, tgt, pr = brute.random_graph(rng, n, 5 * n, [None, 0.05, 0.1, 0.02, 0.3][g], allow_dups=False, allow_loops=False)
        J = [32, 64, 128, 256, 64][g]
        compare_select(n, off, tgt, pr, J, int(rng.integers(0, 2**32)), min(n, 15), t)


def test_select_pool_exhaustion():
    """K = n on a w = 1 graph: the pool empties, the lowest-id vertex not in S is taken (R14, R16)."""
    n = 12
    off = np.arange(n + 1, dtype=np.int32)
    tgt = ((np.arange(n) + 1) % n).astype(np.int32)  # a directed cycle, every vertex reaches all
    compare_select(n, off, tgt, np.ones(n, np.float32), 32, 3, n, 0.05)


def test_select_twice_is_history_free():
    rng = np.random.default_rng(77)
    off, tgt, pr = brute.random_graph(rng, 400, 2000, 0.1)
    im.im_load_csr(400, off, tgt, pr)
    im.im_build_sketches(64, 4)
    a = im.im_select_seeds(8, 0.0)
    b = im.im_select_seeds(8, 0.0)
    assert list(a[0]) == list(b[0]) and list(a[1]) == list(b[1])
