set -x
IM_FIRST_MEM=1 timeout 600 python -m pytest tests -m gpu -x -q -k "test_gpu_parity" > gpurun_out/pytest41.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest41.log
IM_FIRST_MEM=1 IM_TRACE=1 python tools/profile_step.py --config c4 --what build 2>&1 | grep -E "sweep|\{" | head -24 > gpurun_out/trace41_mem.log
IM_TRACE=1 python tools/profile_step.py --config c4 --what build 2>&1 | grep -E "sweep|\{" | head -24 > gpurun_out/trace41.log
IM_FIRST_MEM=1 IM_BENCH_CONFIG=c4 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b41_c4_mem.json 2> gpurun_out/b41_c4_mem.err
IM_BENCH_CONFIG=c4 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b41_c4.json 2> gpurun_out/b41_c4.err
