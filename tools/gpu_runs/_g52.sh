set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "test_gpu_parity or c1 or c2 or c3 or bfs_paths or policy or J64-p0.1-t0.05 or J256-p0.005-t0.05 or slab or shard" > gpurun_out/pytest52.log 2>&1; echo rc=$?; tail -3 gpurun_out/pytest52.log
for c in c4 c3 c2 c1; do IM_BENCH_CONFIG=$c python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b52_$c.json 2> gpurun_out/b52_$c.err; done
