set -x
timeout 1500 python -m pytest tests -m gpu -x -q -k "not c5 and not c4 and not shard and not eval" > gpurun_out/pytest26.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest26.log
IM_BENCH_CONFIG=c4 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b26_c4.json 2> gpurun_out/b26_c4.err; echo bench rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches26_c4.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu26.log 2>&1; echo ncu_launch rc=$?
ncu --set full --import-source on --clock-control none -k regex:'^k_first' --launch-count 4 -o gpurun_out/r02i_first python tools/profile_step.py --config c4 --what build > gpurun_out/ncu26_first.log 2>&1; echo ncu_first rc=$?
