set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv
IM_BENCH_CONFIG=c4 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b22_c4.json 2> gpurun_out/b22_c4.err; echo bench rc=$?; cat gpurun_out/b22_c4.json
ncu --set full --import-source on --clock-control none -k regex:"k_first" --launch-count 4 -o gpurun_out/r02f_first python tools/profile_step.py --config c4 --what build > gpurun_out/ncu22_first.log 2>&1; echo ncu_first rc=$?
ncu --set full --import-source on --clock-control none -k regex:k_bfs_level2 --launch-skip 4 --launch-count 1 -o gpurun_out/r02f_bfs python tools/profile_step.py --config c4 --what step --K 1 > gpurun_out/ncu22_bfs.log 2>&1; echo ncu_bfs rc=$?
ncu --set full --import-source on --clock-control none -k regex:"k_sweep<" --launch-skip 0 --launch-count 1 -o gpurun_out/r02f_push python tools/profile_step.py --config c4 --what build > gpurun_out/ncu22_push.log 2>&1; echo ncu_push rc=$?
