set -x
ncu --set full --clock-control none --import-source on -k regex:"k_bfs_level2|k_bfs_small" --launch-skip 40 -c 4 -o gpurun_out/bfs11_c2 python tools/profile_step.py --config c2 --what step > gpurun_out/ncu11_bfs.log 2>&1; echo ncu rc=$?
IM_BENCH_CONFIG=c2 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b11_c2.json 2>&1; echo c2 rc=$?
IM_BENCH_CONFIG=c1 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b11_c1.json 2>&1; echo c1 rc=$?
IM_PIPELINE=0 IM_BENCH_CONFIG=c1 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b11_c1_nopipe.json 2>&1
IM_TRACE=1 python tools/profile_step.py --config c1 --what step > gpurun_out/trace11_c1.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "bfs or parity and not c5 and not c4" > gpurun_out/pytest11.log 2>&1; echo pytest rc=$?
