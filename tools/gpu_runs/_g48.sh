set -x
IM_LIB=$PWD/variants/batom.so ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_load_c4_batom.csv python tools/profile_step.py --config c4 --what build > gpurun_out/ncu48.log 2>&1; echo rc=$?
IM_LIB=$PWD/variants/batom.so timeout 600 python -m pytest tests -m gpu -x -q -k "test_gpu_parity or c1 or c2 or c3" > gpurun_out/pytest48.log 2>&1; echo rc=$?; tail -3 gpurun_out/pytest48.log
IM_LIB=$PWD/variants/batom.so IM_BENCH_CONFIG=c4 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b48_c4_batom.json 2> gpurun_out/b48_c4.err; echo bench rc=$?
IM_BENCH_CONFIG=c4 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b48_c4.json 2> gpurun_out/b48_c4.err; echo bench rc=$?
