"""im_set_policy and the paper's early-exit variant eps_c > 0 (8(f) f1, reading R22:
synchronous sweeps) on the GPU vs the oracle: registers, sweep counts, full selections with rebuilds;
at C3 size, sampled registers vs the k-hop definition."""
import math

import numpy as np
import pytest

import gen
import oracle
import paper_2105_04023_b200 as im
from tests import brute

pytestmark = pytest.mark.gpu
NAN = float("nan")


@pytest.fixture(autouse=True)
def default_policy():
    im.im_set_policy(NAN, NAN, 0.0)
    yield
    im.im_set_policy(NAN, NAN, 0.0)


def test_policy_validation():
    for args in [(-1.0, NAN, 0.0), (NAN, -0.5, 0.0), (NAN, NAN, -0.1), (NAN, NAN, 1.5), (NAN, NAN, NAN)]:
        with pytest.raises(im.IMError) as e:
            im.im_set_policy(*args)
        assert e.value.code == im.IM_EINVAL


@pytest.mark.parametrize("eps_c", [0.02, 0.1, 0.3, 1.0])
def test_early_exit_build_matches_oracle(eps_c):
    rng = np.random.default_rng(int(eps_c * 100) + 5)
    for g in range(6):
        n = int(rng.integers(200, 2000))
        off, tgt, pr = brute.random_graph(rng, n, int(rng.integers(2 * n, 8 * n)), None if g % 3 == 0 else float(rng.choice([0.05, 0.2, 0.5])))
        J = int(rng.choice([32, 64, 256]))
        seed = int(rng.integers(0, 2**32))
        im.im_set_policy(NAN, NAN, eps_c)
        im.im_load_csr(n, off, tgt, pr)
        im.im_build_sketches(J, seed)
        Mo, st = oracle.simulate(n, off, tgt, pr, J, seed, eps_c=eps_c)
        assert np.array_equal(im.im_get_registers(n, J), Mo), g
        s = im.im_get_stats()
        assert s["last_build_sweeps"] == st["sweeps"] and s["eps_c"] == eps_c


@pytest.mark.parametrize("t", [0.0, 0.05, math.inf])
def test_early_exit_select_matches_oracle(t):
    """Full selection (rebuilds with blocked simulations also stop early) vs the oracle."""
    rng = np.random.default_rng(int(1000 * min(t, 9)) + 17)
    for g in range(4):
        n = int(rng.integers(300, 1500))
        off, tgt, pr = brute.random_graph(rng, n, 5 * n, float(rng.choice([0.05, 0.2])))
        J, seed, K, eps_c = 64, int(rng.integers(0, 2**32)), 12, float(rng.choice([0.02, 0.05]))
        im.im_set_policy(NAN, NAN, eps_c)
        im.im_load_csr(n, off, tgt, pr)
        im.im_build_sketches(J, seed)
        s, sc = im.im_select_seeds(K, t)
        r = oracle.select_seeds(n, off, tgt, pr, J, seed, K, t, want_vis=True, want_final=True, eps_c=eps_c)
        assert list(s) == list(r["seeds"]) and list(sc) == list(r["scores"]), g
        log = im.im_get_step_log(K)
        for a, b in zip(log, r["steps"]):
            assert (a["vertex"], a["score"], a["sigma_count"], a["rebuilt"], a["executed"]) == \
                   (b["vertex"], b["score"], b["sigma_count"], b["rebuilt"], b["executed"])
        assert np.array_equal(im.im_get_registers(n, J), r["M_final"])
        assert np.array_equal(im.reach_bits_to_bool(im.im_get_reach(n, J), J), r["vis"].astype(bool))


def test_policy_thresholds_override_select_threshold():
    """(eps_l, eps_g) = (0.3, 0.01), the paper's pair: im_select_seeds(K, t) ignores t
    and equals im_select_seeds_ex(K, 0.3, 0.01) and the oracle with those thresholds."""
    rng = np.random.default_rng(23)
    n = 800
    off, tgt, pr = brute.random_graph(rng, n, 4000, 0.1)
    J, seed, K = 128, 9, 15
    im.im_load_csr(n, off, tgt, pr)
    im.im_build_sketches(J, seed)
    s_ex, sc_ex = im.im_select_seeds(K, 0.3, 0.01)
    im.im_set_policy(0.3, 0.01, 0.0)
    s_p, sc_p = im.im_select_seeds(K, 123.0)
    r = oracle.select_seeds(n, off, tgt, pr, J, seed, K, 0.3, 0.01)
    assert list(s_p) == list(s_ex) == list(r["seeds"]) and list(sc_p) == list(sc_ex)


def test_policy_change_rebuilds_before_select():
    """Sketches built with eps_c = 0 are rebuilt under the new eps_c before a selection."""
    rng = np.random.default_rng(29)
    n = 1000
    off, tgt, pr = brute.random_graph(rng, n, 6000, 0.2)
    J, seed, K = 64, 4, 5
    im.im_load_csr(n, off, tgt, pr)
    im.im_build_sketches(J, seed)
    im.im_set_policy(NAN, NAN, 0.05)
    s, _ = im.im_select_seeds(K, math.inf)
    r = oracle.select_seeds(n, off, tgt, pr, J, seed, K, math.inf, eps_c=0.05)
    assert list(s) == list(r["seeds"])
    assert im.im_get_stats()["eps_c"] == 0.05


def test_c1_early_exit_full_parity():
    """C1 with the paper's eps_c = 0.02: live oracle, build + K = 10 selection."""
    cfg = gen.CONFIGS["c1"]
    n, off, tgt, pr = gen.workload(cfg)
    im.im_set_policy(NAN, NAN, 0.02)
    im.im_load_csr(n, off, tgt, pr)
    im.im_build_sketches(cfg.J, cfg.salt_seed)
    Mo, st = oracle.simulate(n, off, tgt, pr, cfg.J, cfg.salt_seed, eps_c=0.02)
    assert np.array_equal(im.im_get_registers(n, cfg.J), Mo)
    s, sc = im.im_select_seeds(cfg.K, cfg.t)
    r = oracle.select_seeds(n, off, tgt, pr, cfg.J, cfg.salt_seed, cfg.K, cfg.t, eps_c=0.02)
    assert list(s) == list(r["seeds"]) and list(sc) == list(r["scores"])


def test_c3_early_exit_sampled_khop():
    """C3 (4M vertices, J = 256) with eps_c = 0.02: the build stops after s sweeps and every sampled
    register equals the max init register within s hops (the synchronous-schedule definition)."""
    cfg = gen.CONFIGS["c3"]
    from tests.test_gpu_configs import cached_graph

    n, off, tgt = cached_graph(cfg.graph)
    pr = np.full(len(tgt), cfg.p, np.float32)
    im.im_set_policy(NAN, NAN, 0.02)
    im.im_load_csr(n, off, tgt, pr)
    im.im_build_sketches(cfg.J, cfg.salt_seed)
    hops = im.im_get_stats()["last_build_sweeps"]
    assert hops >= 1
    rng = np.random.default_rng(31)
    us = rng.integers(0, n, 300).astype(np.int32)
    js = rng.integers(0, cfg.J, 300).astype(np.int32)
    rows = im.im_get_register_rows(us, cfg.J)
    want = oracle.khop_register(n, off, tgt, pr, cfg.J, cfg.salt_seed, hops, us, js)
    assert np.array_equal(rows[np.arange(300), js], want)
    full = oracle.reach_register(n, off, tgt, pr, cfg.J, cfg.salt_seed, us, js)
    assert (want <= full).all()
    s, sc = im.im_select_seeds(cfg.K, cfg.t)
    assert len(set(s.tolist())) == cfg.K and all(np.diff(sc) >= 0)
