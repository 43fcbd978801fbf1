# round-2 capture: smoke, all GPU tests, bench lines C4 (+e2e, cpu_baseline), C1-C3, reference arm, launch list,
# DRAM traffic of one step (application replay), ncu full of the top kernels, C5 corners
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
( time timeout 3000 python -m pytest tests -m gpu -x -q --durations=15 -rx ) > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo bench rc=$?; cat gpurun_out/bench_c4.json
for c in c1 c2 c3; do python bench.py --config $c --steps 5 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench $c rc=$?; done
python bench.py --impl reference --steps 1 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench.log 2>&1; echo ncu_launch rc=$?
ncu --replay-mode application --app-replay-mode relaxed --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum --clock-control none --csv --log-file gpurun_out/dram.csv python tools/profile_step.py --config c4 --what step > gpurun_out/ncu_dram.log 2>&1; echo ncu_dram rc=$?
ncu --set full --import-source on --clock-control none -k regex:'^k_first' --launch-count 4 -o gpurun_out/ncu_first python tools/profile_step.py --config c4 --what build > gpurun_out/ncu_first.log 2>&1; echo ncu_first rc=$?
ncu --set full --import-source on --clock-control none -k regex:'^k_sweep$' --launch-count 1 -o gpurun_out/ncu_push python tools/profile_step.py --config c4 --what build > gpurun_out/ncu_push.log 2>&1; echo ncu_push rc=$?
ncu --set full --import-source on --clock-control none -k regex:'^k_bfs_level2$' --launch-skip 4 --launch-count 1 -o gpurun_out/ncu_bfs python tools/profile_step.py --config c4 --what step --K 1 > gpurun_out/ncu_bfs.log 2>&1; echo ncu_bfs rc=$?
python tools/sweep_c5.py --points all --reps 3 > gpurun_out/c5_grid.jsonl 2> gpurun_out/c5_grid.txt; echo c5 rc=$?
