"""Independent Monte-Carlo influence evaluator (reading R23): im_evaluate vs the
oracle's sample-then-diffuse definition, bit-exact counts, small graphs and C3 / C4 at full size."""
import numpy as np
import pytest

import gen
import oracle
import paper_2105_04023_b200 as im
from tests import brute

pytestmark = pytest.mark.gpu


def test_evaluate_validation():
    n = 10
    off, tgt, pr = np.arange(11, dtype=np.int32), (np.arange(1, 11) % 10).astype(np.int32), np.full(10, 0.5, np.float32)
    im.im_load_csr(n, off, tgt, pr)
    for seeds, R, r0 in [([0, 10], 32, 0), ([-1], 32, 0), ([0], 48, 0), ([0], 0, 0), ([0], 32, -1)]:
        with pytest.raises(im.IMError) as e:
            im.im_evaluate(seeds, 1, R, r0)
        assert e.value.code == im.IM_EINVAL
    assert len(im.im_evaluate([], 1, 32)) == 0


@pytest.mark.parametrize("R,r0", [(32, 0), (96, 37), (1024, 5)])
def test_evaluate_small_graphs_match_oracle(R, r0):
    rng = np.random.default_rng(R + r0)
    for g in range(5):
        n = int(rng.integers(50, 3000))
        p = None if g % 2 else float(rng.choice([0.02, 0.1, 0.4]))
        off, tgt, pr = brute.random_graph(rng, n, int(rng.integers(n, 6 * n)), p)
        seeds = rng.integers(0, n, int(rng.integers(1, 12))).astype(np.int32)
        seed = int(rng.integers(0, 2**63))
        im.im_load_csr(n, off, tgt, pr)
        got = im.im_evaluate(seeds, seed, R, r0)
        want = oracle.mc_influence(n, off, tgt, pr, seeds, seed, r0, R)
        assert np.array_equal(got, want), (g, got, want)


def test_evaluate_sample_ranges_add_up():
    rng = np.random.default_rng(3)
    n = 2000
    off, tgt, pr = brute.random_graph(rng, n, 12000, 0.15)
    seeds = np.array([5, 77, 1500], np.int32)
    im.im_load_csr(n, off, tgt, pr)
    a = im.im_evaluate(seeds, 9, 640)
    b = im.im_evaluate(seeds, 9, 320) + im.im_evaluate(seeds, 9, 320, r0=320)
    assert np.array_equal(a, b) and all(np.diff(a) >= 0)


def test_evaluate_c3_full_size():
    """C3 (Chung-Lu 4M / 67.9M, p = 0.01): 32 fresh samples of the K = 50 selection's seeds."""
    cfg = gen.CONFIGS["c3"]
    from tests.test_gpu_configs import cached_graph

    n, off, tgt = cached_graph(cfg.graph)
    pr = np.full(len(tgt), cfg.p, np.float32)
    im.im_load_csr(n, off, tgt, pr)
    im.im_build_sketches(cfg.J, cfg.salt_seed)
    s, sc = im.im_select_seeds(cfg.K, cfg.t)
    got = im.im_evaluate(s[:10], 2024, 32)
    want = oracle.mc_influence(n, off, tgt, pr, s[:10], 2024, 0, 32)
    assert np.array_equal(got, want)
    # fresh samples vs the sketches' own samples: same expectation (sigma ~ independent estimate)
    mc = im.im_evaluate(s, 2024, 512)[-1] / 512
    assert abs(mc - sc[-1]) / sc[-1] < 0.1


def test_evaluate_c4_sampled():
    """C4 (RMAT-24, 520.8M edges): 32 fresh samples of 5 seeds vs the oracle at full size."""
    cfg = gen.CONFIGS["c4"]
    n, off, tgt, pr = gen.workload(cfg)
    im.im_load_csr(n, off, tgt, pr)
    deg = np.diff(off)
    seeds = np.argsort(deg)[-5:][::-1].astype(np.int32)
    got = im.im_evaluate(seeds, 77, 32, r0=1000)
    want = oracle.mc_influence(n, off, tgt, pr, seeds, 77, 1000, 32)
    assert np.array_equal(got, want)
