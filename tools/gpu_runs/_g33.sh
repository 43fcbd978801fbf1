set -x
IM_SLAB_MIN_M=0 timeout 1500 python -m pytest tests -m gpu -x -q -k "not c5 and not c4 and not shard_mp and not eval" > gpurun_out/pytest33_slab.log 2>&1; echo pytest rc=$?; tail -5 gpurun_out/pytest33_slab.log
timeout 900 python -m pytest tests -m gpu -x -q -k "c3_parity or c2_parity" > gpurun_out/pytest33.log 2>&1; echo pytest rc=$?; tail -5 gpurun_out/pytest33.log
for sp in 3 4 5; do
IM_SLAB_PASSES=$sp IM_BENCH_CONFIG=c4 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b33_c4_sp$sp.json 2> gpurun_out/b33_c4_sp$sp.err; echo bench rc=$?
done
IM_BENCH_CONFIG=c3 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b33_c3.json 2>&1
IM_TRACE=1 python tools/profile_step.py --config c4 --what build 2>&1 | grep "sweep [1-4] " > gpurun_out/trace33.log
ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none -c 4000 --csv --log-file gpurun_out/launches33_c4.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu33.log 2>&1; echo ncu_launch rc=$?
