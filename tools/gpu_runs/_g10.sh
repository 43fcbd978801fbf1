set -x
timeout 1200 python -m pytest tests -m gpu -x -q -k "not c5 and not c4" > gpurun_out/pytest10.log 2>&1; echo pytest rc=$?
for c in c4 c2 c1 c3; do
IM_BENCH_CONFIG=$c python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b10_$c.json 2> gpurun_out/b10_$c.err; echo bench $c rc=$?
done
IM_PIPELINE=0 IM_BENCH_CONFIG=c2 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b10_c2_nopipe.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches10_c2.csv python tools/profile_step.py --config c2 --what step > gpurun_out/ncu10_c2.log 2>&1; echo ncu c2 rc=$?
ncu --replay-mode application --app-replay-mode relaxed --app-replay-match name --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum --clock-control none --csv --log-file gpurun_out/dram10.csv python tools/profile_step.py --config c4 --what step > gpurun_out/ncu10_dram.log 2>&1; echo ncu_dram rc=$?
