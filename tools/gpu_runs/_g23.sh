set -x
timeout 1500 python -m pytest tests -m gpu -x -q -k "not c5 and not c4" > gpurun_out/pytest23.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest23.log
for tr in 1 0; do
IM_THREAD_ROWS=$tr IM_BENCH_CONFIG=c4 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b23_c4_tr$tr.json 2> gpurun_out/b23_c4_tr$tr.err; echo bench rc=$?
done
IM_BENCH_CONFIG=c3 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b23_c3.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches23_c4.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu23.log 2>&1; echo ncu_launch rc=$?
