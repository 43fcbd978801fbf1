set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "not c5 and not c4 and not eval" > gpurun_out/pytest8.log 2>&1; echo pytest rc=$?
IM_BENCH_CONFIG=c4 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b8_c4.json 2> gpurun_out/b8_c4.err; echo bench rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches8_c4.csv python tools/profile_step.py --config c4 --what step > gpurun_out/ncu8_c4.log 2>&1; echo ncu c4 rc=$?
