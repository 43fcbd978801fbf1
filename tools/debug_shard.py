"""Compare a sharded selection (world ranks as threads, or world=1 with an identity hook) with the
unsharded one, step by step (diagnostic)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2105_04023_b200 as im  # noqa: E402
from tests import brute  # noqa: E402
from tests.test_gpu_shard import run_sharded, unsharded  # noqa: E402

J, world, eps = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])
rng = np.random.default_rng(J + world)
n = 300
off, tgt, pr = brute.random_graph(rng, n, 1500)
K, seed = 12, 5
ref = unsharded(n, off, tgt, pr, J, seed, K, eps)
for rep in range(2):
    out, calls = run_sharded(world, n, off, tgt, pr, J, seed, K, eps)
    print("rep", rep, "calls", calls)
    for k in range(K):
        a = ref["log"][k]
        row = [(a["vertex"], a["score"], a["sigma_count"], a["rebuilt"])]
        for o in out:
            b = o["log"][k]
            row.append((b["vertex"], b["score"], b["sigma_count"], b["rebuilt"]))
        print(k, "OK " if len(set(row)) == 1 else "BAD", row)
    print("est equal", [bool(np.array_equal(o["est"], ref["est"])) for o in out])
    for o in out:
        print({k: o["stats"][k] for k in ("J", "J_total", "j0", "argmax_full", "argmax_lazy", "rebuilds")})
