set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "J1024-p0.005 or J1024-p0.01-t0.3 or estimate or test_constant_w" -rx > gpurun_out/pytest60.log 2>&1; echo rc=$?; tail -5 gpurun_out/pytest60.log
python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo bench rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench.log 2>&1; echo ncu_launch rc=$?
