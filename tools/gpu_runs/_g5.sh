set -x
IM_BENCH_CONFIG=c4 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b5_c4.json 2> gpurun_out/b5_c4.err; echo bench rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_scatter -c 1 -o gpurun_out/scatter5 python tools/profile_step.py --config c4 --what build > gpurun_out/ncu5_scatter.log 2>&1; echo ncu1 rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches5_c4.csv python tools/profile_step.py --config c4 --what step > gpurun_out/ncu5_c4.log 2>&1; echo ncu c4 rc=$?
timeout 900 python -m pytest tests -m gpu -x -q -k "parity and not c5 and not c4" > gpurun_out/pytest5.log 2>&1; echo pytest rc=$?
