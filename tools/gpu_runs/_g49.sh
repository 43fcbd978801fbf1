set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "test_gpu_parity or c1 or c2 or c3 or bfs_paths or J64-p0.1-t0.05 or J256-p0.005-t0.05 or policy" > gpurun_out/pytest49.log 2>&1; echo rc=$?; tail -3 gpurun_out/pytest49.log
IM_BENCH_CONFIG=c4 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b49_c4.json 2> gpurun_out/b49_c4.err; echo bench rc=$?
for c in c2 c3; do IM_BENCH_CONFIG=$c python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b49_$c.json 2> gpurun_out/b49_$c.err; done
