set -x
timeout 1500 python -m pytest tests -m gpu -x -q -k "not c5 and not c4 and not shard and not eval" > gpurun_out/pytest28.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest28.log
IM_BENCH_CONFIG=c4 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b28_c4.json 2> gpurun_out/b28_c4.err; echo bench rc=$?
for v in lb0 bps6 bps8; do
IM_LIB=$PWD/variants/$v.so IM_BENCH_CONFIG=c4 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b28_c4_$v.json 2> gpurun_out/b28_c4_$v.err; echo bench rc=$?
done
IM_BENCH_CONFIG=c3 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b28_c3.json 2>&1
IM_BENCH_CONFIG=c2 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b28_c2.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches28_c4.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu28.log 2>&1; echo ncu_launch rc=$?
