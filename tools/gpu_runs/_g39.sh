set -x
timeout 1500 python -m pytest tests -m gpu -x -q -k "not c5 and not c4 and not shard_mp and not eval and not slab" > gpurun_out/pytest39.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest39.log
timeout 900 python -m pytest tests -m gpu -x -q -k "J64-p0.1-t0.05 or J128-p0.1-t0.05 or J256-p0.1-t0.05" > gpurun_out/pytest39b.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest39b.log
IM_TRACE=1 python tools/profile_step.py --config c3 --what build --J 1024 --p 0.1 2>&1 | grep -E "sweep|\{" | head -8 > gpurun_out/trace39.log
IM_TRACE=1 python tools/profile_step.py --config c3 --what build --J 512 --p 0.1 2>&1 | grep -E "sweep|\{" | head -8 > gpurun_out/trace39b.log
IM_BENCH_CONFIG=c4 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b39_c4.json 2> gpurun_out/b39_c4.err; echo bench rc=$?
IM_BENCH_CONFIG=c2 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b39_c2.json 2>&1
