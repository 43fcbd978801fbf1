set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "parity and not c5 and not c4" > gpurun_out/pytest6.log 2>&1; echo pytest rc=$?
IM_BENCH_CONFIG=c4 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b6_c4.json 2> gpurun_out/b6_c4.err; echo bench rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches6_c4.csv python tools/profile_step.py --config c4 --what step > gpurun_out/ncu6_c4.log 2>&1; echo ncu c4 rc=$?
ncu --set full --clock-control none --import-source on -k regex:"k_part|k_place|k_first_big|k_rows_big" -c 6 -o gpurun_out/prep6 python tools/profile_step.py --config c4 --what build > gpurun_out/ncu6_prep.log 2>&1; echo ncu2 rc=$?
