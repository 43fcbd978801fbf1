"""Build an experiment copy of the library with extra nvcc defines (A/B runs via IM_LIB=<path>).

    python tools/build_variant.py variants/ep2.so -DBFS_EP=2 -DBFS_MINB=1
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2105_04023_b200 import _build  # noqa: E402

out, defs = sys.argv[1], sys.argv[2:]
os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
cmd = [os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc"), *[f for f in _build.NVCC_FLAGS if f not in ("-Xptxas", "-v")], *defs,
       "-o", out, *[os.path.join(_build.CSRC, s) for s in _build.SOURCES]]
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stdout + r.stderr)
print(out)
