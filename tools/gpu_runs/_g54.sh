set -x
IM_LIB=$PWD/variants/bfsc.so timeout 900 python -m pytest tests -m gpu -x -q -k "test_gpu_parity or c1 or c2 or c3 or bfs_paths or eval or J64-p0.1-t0.05 or J128-p0.01-t0.05" > gpurun_out/pytest54.log 2>&1; echo rc=$?; tail -3 gpurun_out/pytest54.log
for c in c4 c3 c2; do IM_LIB=$PWD/variants/bfsc.so IM_BENCH_CONFIG=$c python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b54_${c}_bfsc.json 2> gpurun_out/b54_$c.err; done
IM_BENCH_CONFIG=c4 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b54_c4.json 2> gpurun_out/b54_c4.err
