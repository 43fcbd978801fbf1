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
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


_graphs = {}


def cached_graph(name):
    if name not in _graphs:
        _graphs[name] = gen.graph(name)
    return _graphs[name]


def golden(tag):
    p = os.path.join(GOLDEN, f"{tag}_oracle.json")
    return json.load(open(p)) if os.path.exists(p) else None


def reach_words_abi(n, J):
    return im.im_get_reach(n, J)


def test_c1_full_parity_live_oracle():
    cfg = gen.CONFIGS["c1"]
    n, off, tgt, pr = gen.workload(cfg)
    g = golden("c1")
    assert g["graph_sha256"] == sha(off, tgt, pr)
    im.im_load_csr(n, off, tgt, pr)
    im.im_build_sketches(cfg.J, cfg.salt_seed)
    M = im.im_get_registers(n, cfg.J)
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
    rows = im.im_get_register_rows(us, J)
    want = oracle.reach_register(n, off, tgt, pr, J, seed, us, js)
    got = rows[np.arange(n_samples), js]
    assert np.array_equal(got, want), np.nonzero(got != want)


def test_c2_parity():
    cfg = gen.CONFIGS["c2"]
    n, off, tgt, pr = gen.workload(cfg)
    im.im_load_csr(n, off, tgt, pr)
    im.im_build_sketches(cfg.J, cfg.salt_seed)
    g = golden("c2")
    if g is not None and "first_build" in g:
        assert g["graph_sha256"] == sha(off, tgt, pr)
        M = im.im_get_registers(n, cfg.J)
        assert sha(M) == g["first_build"]["registers_sha256"]
        sr = g["first_build"]["sample_rows"]
        assert np.array_equal(M[sr["vertices"]], np.array(sr["rows"], np.uint8))
    sampled_register_check(n, off, tgt, pr, cfg.J, cfg.salt_seed, 300)
    s, sc = im.im_select_seeds(cfg.K, cfg.t)
    # sigma of the GPU's own seeds, recomputed by the oracle's BFS definition at full size
    cnt = oracle.seed_sigma(n, off, tgt, pr, cfg.J, cfg.salt_seed, s)
    assert list(sc) == list(cnt / cfg.J)
    if g is not None and "select" in g:
        assert list(s) == g["select"]["seeds"]
        assert [x["rebuilt"] for x in im.im_get_step_log(cfg.K)] == g["select"]["rebuilt"]
        assert sha(reach_words_abi(n, cfg.J)) == g["select"]["reach_sha256"]


def sampled_seed_reach_check(n, off, tgt, pr, J, seed, seeds, sims):
    """Per-simulation |R_G(S)| of the GPU's seed set vs the oracle's BFS definition, for a few simulations."""
    vis = im.reach_bits_to_bool(im.im_get_reach(n, J), J)
    want = oracle.seed_reach_per_sim(n, off, tgt, pr, J, seed, sims, seeds)
    assert [int(vis[:, j].sum()) for j in sims] == list(want[:, -1])


def test_c3_parity():
    """C3 (Chung-Lu, 4M / 67.9M, p = 0.01, J = 256): first-build registers vs the oracle's digest,
    sampled registers vs the reach-max definition, K = 50 selection: sigma of every step vs the
    step log, per-simulation reach of the seed set vs the oracle's BFS."""
    cfg = gen.CONFIGS["c3"]
    n, off, tgt = cached_graph(cfg.graph)
    pr = np.full(len(tgt), cfg.p, np.float32)
    im.im_load_csr(n, off, tgt, pr)
    im.im_build_sketches(cfg.J, cfg.salt_seed)
    g = golden("c3")
    if g is not None:
        assert g["graph_sha256"] == sha(off, tgt, pr)
        M = im.im_get_registers(n, cfg.J)
        assert sha(M) == g["first_build"]["registers_sha256"]
        del M
    sampled_register_check(n, off, tgt, pr, cfg.J, cfg.salt_seed, 300, rng_seed=3)
    s, sc = im.im_select_seeds(cfg.K, cfg.t)
    assert len(set(s.tolist())) == cfg.K and all(np.diff(sc) >= 0)
    log = im.im_get_step_log(cfg.K)
    assert [x["sigma_count"] / cfg.J for x in log] == list(sc)
    sampled_seed_reach_check(n, off, tgt, pr, cfg.J, cfg.salt_seed, s, [0, 97, 255])


def test_c4_parity():
    """C4 (RMAT-24, 16.8M / 520.8M, p = 0.005, J = 512): sampled registers of the first build vs
    the reach-max definition (and the oracle's digest when tests/golden/c4_oracle.json exists),
    K = 50 selection, per-simulation reach of the seed set vs the oracle's BFS."""
    cfg = gen.CONFIGS["c4"]
    n, off, tgt, pr = gen.workload(cfg)
    im.im_load_csr(n, off, tgt, pr)
    im.im_build_sketches(cfg.J, cfg.salt_seed)
    g = golden("c4")
    if g is not None and "first_build" in g:
        assert g["graph_sha256"] == sha(off, tgt, pr)
        sr = g["first_build"]["sample_rows"]
        assert np.array_equal(im.im_get_register_rows(np.array(sr["vertices"], np.int32), cfg.J), np.array(sr["rows"], np.uint8))
        assert sha(im.im_get_registers(n, cfg.J)) == g["first_build"]["registers_sha256"]
    sampled_register_check(n, off, tgt, pr, cfg.J, cfg.salt_seed, 200, rng_seed=4)
    s, sc = im.im_select_seeds(cfg.K, cfg.t)
    assert len(set(s.tolist())) == cfg.K and all(np.diff(sc) >= 0)
    sampled_seed_reach_check(n, off, tgt, pr, cfg.J, cfg.salt_seed, s, [5, 300])


@pytest.mark.parametrize("J,p,t", [(64, 0.005, 0.01), (1024, 0.1, 0.3), (128, 0.01, 0.05), (512, 0.1, 0.01)])
def test_c5_grid_points(J, p, t):
    """C5 grid corners on the C3 graph (J x p x t, K = 100): sampled registers of the first build,
    the selection's invariants and the per-simulation reach of its seeds (J = 1024 / p = 0.1 drives
    128-simulation windows through the warp-cooperative paths)."""
    n, off, tgt = cached_graph("cl4m")
    pr = np.full(len(tgt), p, np.float32)
    im.im_load_csr(n, off, tgt, pr)
    im.im_build_sketches(J, 1)
    sampled_register_check(n, off, tgt, pr, J, 1, 100, rng_seed=J)
    s, sc = im.im_select_seeds(100, t)
    assert len(set(s.tolist())) == 100 and all(np.diff(sc) >= 0)
    sampled_seed_reach_check(n, off, tgt, pr, J, 1, s, [0, J - 1])
