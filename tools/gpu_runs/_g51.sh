set -x
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_pscatter|k_pcount|k_place|k_part' -c 8 --csv --log-file gpurun_out/launches_load_c4_g51.csv python tools/profile_step.py --config c4 --what build > gpurun_out/ncu51.log 2>&1; echo rc=$?
timeout 900 python -m pytest tests -m gpu -x -q -k "test_gpu_parity or c1 or c2 or c3" > gpurun_out/pytest51.log 2>&1; echo rc=$?; tail -3 gpurun_out/pytest51.log
IM_BENCH_CONFIG=c4 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b51_c4.json 2> gpurun_out/b51_c4.err; echo bench rc=$?
