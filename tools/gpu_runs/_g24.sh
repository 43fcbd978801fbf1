set -x
timeout 1500 python -m pytest tests -m gpu -x -q -k "not c5 and not c4 and not shard and not eval" > gpurun_out/pytest24.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest24.log
IM_BENCH_CONFIG=c4 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b24_c4.json 2> gpurun_out/b24_c4.err; echo bench rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches24_c4.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu24.log 2>&1; echo ncu_launch rc=$?
ncu --set full --import-source on --clock-control none -k regex:'^k_first$' --launch-count 2 -o gpurun_out/r02g_first python tools/profile_step.py --config c4 --what build > gpurun_out/ncu24_first.log 2>&1; echo ncu_first rc=$?
ncu --set full --import-source on --clock-control none -k regex:'^k_sweep$' --launch-count 1 -o gpurun_out/r02g_push python tools/profile_step.py --config c4 --what build > gpurun_out/ncu24_push.log 2>&1; echo ncu_push rc=$?
