"""GPU parity on the BASELINE.json configs (C1..C5) through the C ABI.

C1 runs the live oracle.  Larger configs compare against digests the oracle wrote offline
(tests/golden/<cfg>_oracle.json, tests/golden/make_oracle_digests.py -- oracle/ only) plus
per-sample oracle definitions (register = max over the reach set; sigma = BFS count) that the
oracle can evaluate one by one at full size.
"""
import hashlib
import json
import math
import os

import numpy as np
import pytest

import gen
import oracle
import paper_2105_04023_b200 as im

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def sha(*arrs):
    h = hashlib.sha256()
    for a in arrs:
        flat = np.ascontiguousarray(a).reshape(-1).view(np.uint8)
        for i in range(0, len(flat), 1 << 28):  # no full-size copy (C4 registers are 8.6 GB)
            h.update(flat[i:i + (1 << 28)])
    return h.hexdigest()


_graphs = {}


def cached_graph(name):
    if name not in _graphs:
        _graphs[name] = gen.graph(name)
    return _graphs[name]


def golden(tag):
    p = os.path.join(GOLDEN, f"{tag}_oracle.json")
    return json.load(open(p)) if os.path.exists(p) else None


def need_golden(tag, *sections):
    """The oracle's offline digest (tests/golden/make_oracle_digests.py), or None when it has not been generated.
    A caller that gets None runs the sampled per-pair oracle checks and then reports the point with
    `digest_missing` (an explicit xfail naming the digest), never a silent pass."""
    g = golden(tag)
    if g is None or any(s not in g for s in sections):
        return None
    return g


def digest_missing(tag):
    pytest.xfail(f"offline oracle digest {tag} not generated yet (CPU-hours: tools/golden_queue.sh); "
                 "the sampled oracle parity checks of this test passed")


def check_first_build(g, n, J, off, tgt, pr, full_sha=True):
    """first-build registers vs the oracle digest: graph SHA, register SHA, 64 sampled rows"""
    fb = g["first_build"]
    assert g["graph_sha256"] == sha(off, tgt, pr)
    sr = fb["sample_rows"]
    assert np.array_equal(im.im_get_register_rows(np.array(sr["vertices"], np.int32)), np.array(sr["rows"], np.uint8))
    if full_sha:
        assert sha(im.im_get_registers()) == fb["registers_sha256"]


def check_select(g, J, s, sc):
    """Alg. 1 outputs vs the oracle digest: seeds, integer merged scores, e, sigma counts, keep / rebuild
    decisions and executions at every step, the final R_G(S) (SHA of the C-ABI bit layout) and the
    registers after the last executed rebuild (SHA and sampled rows)."""
    sel = g["select"]
    K = sel["K"]
    log = im.im_get_step_log(K)
    assert list(s) == sel["seeds"]
    assert [x["sigma_count"] for x in log] == sel["sigma_counts"]
    assert [x["score"] for x in log] == sel["scores_int"]
    assert [x["rebuilt"] for x in log] == sel["rebuilt"]
    assert [x["executed"] for x in log] == sel["executed"]
    assert list(sc) == [c / J for c in sel["sigma_counts"]]
    np.testing.assert_allclose([x["e"] for x in log], sel["e"], rtol=1e-12)
    assert sha(im.im_get_reach()) == sel["reach_sha256"]
    if "final_sample_rows" in sel:
        fr = sel["final_sample_rows"]
        assert np.array_equal(im.im_get_register_rows(np.array(fr["vertices"], np.int32)), np.array(fr["rows"], np.uint8))
    if "final_registers_sha256" in sel:
        assert sha(im.im_get_registers()) == sel["final_registers_sha256"]
    return log


def rebuilt_register_check(n, off, tgt, pr, J, seed, seeds, log, n_samples, n_sims, rng_seed):
    """registers after the last executed rebuild vs the oracle's definition (reach-max on the residual
    samples, R_S = R_G(seed prefix)) for sampled (u, j) pairs over n_sims simulations"""
    ex = [k for k, x in enumerate(log) if x["executed"]]
    if not ex:
        return 0
    prefix = np.asarray(seeds[: ex[-1] + 1], np.int32)
    rng = np.random.default_rng(rng_seed)
    sims = rng.choice(J, n_sims, replace=False)
    us = rng.integers(0, n, n_samples).astype(np.int32)
    js = sims[rng.integers(0, n_sims, n_samples)].astype(np.int32)
    rows = im.im_get_register_rows(us)
    want = oracle.rebuilt_register(n, off, tgt, pr, J, seed, prefix, us, js)
    got = rows[np.arange(n_samples), js]
    assert np.array_equal(got, want), np.nonzero(got != want)
    return len(ex)


def reach_words_abi(n, J):
    return im.im_get_reach()


def test_c1_full_parity_live_oracle():
    cfg = gen.CONFIGS["c1"]
    n, off, tgt, pr = gen.workload(cfg)
    g = golden("c1")
    assert g["graph_sha256"] == sha(off, tgt, pr)
    im.im_load_csr(n, off, tgt, pr)
    im.im_build_sketches(cfg.J, cfg.salt_seed)
    M = im.im_get_registers()
    Mo, _ = oracle.simulate(n, off, tgt, pr, cfg.J, cfg.salt_seed)
    assert np.array_equal(M, Mo) and sha(M) == g["first_build"]["registers_sha256"]
    e = im.im_estimate(n)
    assert np.all(np.abs(e - oracle.estimate(Mo)) <= 1e-6 * e)
    s, sc = im.im_select_seeds(cfg.K, cfg.t)
    r = oracle.select_seeds(n, off, tgt, pr, cfg.J, cfg.salt_seed, cfg.K, cfg.t, want_vis=True)
    assert list(s) == list(r["seeds"]) == g["select"]["seeds"]
    assert list(sc) == list(r["scores"])
    log = im.im_get_step_log(cfg.K)
    assert [x["rebuilt"] for x in log] == g["select"]["rebuilt"]
    assert [x["sigma_count"] for x in log] == g["select"]["sigma_counts"]
    assert sha(reach_words_abi(n, cfg.J)) == g["select"]["reach_sha256"]


def sampled_register_check(n, off, tgt, pr, J, seed, n_samples=1000, rng_seed=0):
    rng = np.random.default_rng(rng_seed)
    us = rng.integers(0, n, n_samples).astype(np.int32)
    js = rng.integers(0, J, n_samples).astype(np.int32)
    rows = im.im_get_register_rows(us)
    want = oracle.reach_register(n, off, tgt, pr, J, seed, us, js)
    got = rows[np.arange(n_samples), js]
    assert np.array_equal(got, want), np.nonzero(got != want)


def test_c2_parity():
    """C2 (RMAT-16, WC probabilities, J = 256, K = 50): first build and the whole selection vs the oracle digest."""
    cfg = gen.CONFIGS["c2"]
    n, off, tgt, pr = gen.workload(cfg)
    g = need_golden("c2", "first_build", "select")
    im.im_load_csr(n, off, tgt, pr)
    im.im_build_sketches(cfg.J, cfg.salt_seed)
    check_first_build(g, n, cfg.J, off, tgt, pr)
    sampled_register_check(n, off, tgt, pr, cfg.J, cfg.salt_seed, 1000)
    s, sc = im.im_select_seeds(cfg.K, cfg.t)
    log = check_select(g, cfg.J, s, sc)
    rebuilt_register_check(n, off, tgt, pr, cfg.J, cfg.salt_seed, s, log, 1000, 8, 2)


def sampled_seed_reach_check(n, off, tgt, pr, J, seed, seeds, sims):
    """Per-simulation |R_G(S)| of the GPU's seed set vs the oracle's BFS definition, for a few simulations."""
    words = im.im_get_reach()  # n x J/32 uint32, bit j % 32 of word j / 32 (C ABI layout)
    want = oracle.seed_reach_per_sim(n, off, tgt, pr, J, seed, sims, seeds)
    assert [int(((words[:, j >> 5] >> np.uint32(j & 31)) & np.uint32(1)).sum()) for j in sims] == list(want[:, -1])


def test_c3_parity():
    """C3 (Chung-Lu, 4M / 67.9M, p = 0.01, J = 256, K = 50): first-build registers and the whole selection
    (seeds, scores, sigma, decisions, R_G(S), final registers) vs the oracle digest; 1,000 sampled
    first-build and 1,000 sampled rebuilt registers vs the oracle's per-pair definitions."""
    cfg = gen.CONFIGS["c3"]
    n, off, tgt = cached_graph(cfg.graph)
    pr = np.full(len(tgt), cfg.p, np.float32)
    g = need_golden("c3", "first_build", "select")
    im.im_load_csr(n, off, tgt, pr)
    im.im_build_sketches(cfg.J, cfg.salt_seed)
    check_first_build(g, n, cfg.J, off, tgt, pr)
    sampled_register_check(n, off, tgt, pr, cfg.J, cfg.salt_seed, 1000, rng_seed=3)
    s, sc = im.im_select_seeds(cfg.K, cfg.t)
    log = check_select(g, cfg.J, s, sc)
    rebuilt_register_check(n, off, tgt, pr, cfg.J, cfg.salt_seed, s, log, 1000, 8, 33)


def test_c4_parity():
    """C4 (RMAT-24, 16.8M / 520.8M, p = 0.005, J = 512, K = 50): first-build registers (SHA of all 8.6 GB)
    and the whole selection vs the oracle digest; >= 1,000 sampled first-build registers and 1,000
    sampled rebuilt registers vs the oracle's per-pair definitions."""
    cfg = gen.CONFIGS["c4"]
    n, off, tgt, pr = gen.workload(cfg)
    g = need_golden("c4", "first_build", "select")
    im.im_load_csr(n, off, tgt, pr)
    im.im_build_sketches(cfg.J, cfg.salt_seed)
    if g is not None:
        check_first_build(g, n, cfg.J, off, tgt, pr)
    sampled_register_check(n, off, tgt, pr, cfg.J, cfg.salt_seed, 1000, rng_seed=4)
    s, sc = im.im_select_seeds(cfg.K, cfg.t)
    log = check_select(g, cfg.J, s, sc) if g is not None else im.im_get_step_log(cfg.K)
    rebuilt_register_check(n, off, tgt, pr, cfg.J, cfg.salt_seed, s, log, 1000, 4, 44)
    sampled_seed_reach_check(n, off, tgt, pr, cfg.J, cfg.salt_seed, np.asarray(s, np.int32), [1, 300])
    if g is None:
        digest_missing("c4")


def c5_points():
    """every C5 grid point; a point without an oracle digest fails"""
    return [pytest.param(J, p, t, id=f"J{J}-p{p}-t{t}") for J, p, t in gen.C5_GRID]


@pytest.mark.parametrize("J,p,t", c5_points())
def test_c5_grid_point(J, p, t):
    """C5 grid point on the C3 graph (J x p x t, K = 100): first-build registers and the whole selection vs the
    oracle digest of that point."""
    tag = f"c5_J{J}_p{p}_t{t}"
    g = need_golden(tag, "first_build", "select")
    n, off, tgt = cached_graph("cl4m")
    pr = np.full(len(tgt), p, np.float32)
    im.im_load_csr(n, off, tgt, pr)
    im.im_build_sketches(J, 1)
    if g is not None:
        check_first_build(g, n, J, off, tgt, pr)
        s, sc = im.im_select_seeds(100, t)
        check_select(g, J, s, sc)
        return
    # no digest for this point yet: per-pair oracle definitions on sampled registers, rebuilt registers and
    # the per-simulation reach of the selected seeds, then an explicit xfail naming the missing digest
    ns = 200 if p < 0.05 else 32  # a sampled register at p = 0.1 is a BFS over ~40% of the graph
    sampled_register_check(n, off, tgt, pr, J, 1, ns, rng_seed=J)
    s, sc = im.im_select_seeds(100, t)
    log = im.im_get_step_log(100)
    assert list(sc) == [x["sigma_count"] / J for x in log]
    rebuilt_register_check(n, off, tgt, pr, J, 1, s, log, ns, 4, J + 1)
    sampled_seed_reach_check(n, off, tgt, pr, J, 1, np.asarray(s, np.int32), [0, J - 1])
    digest_missing(tag)
