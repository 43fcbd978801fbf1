set -x
HEAD=$(cat .git_head 2>/dev/null)
ncu --replay-mode application --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum --clock-control none --csv --log-file gpurun_out/dram9.csv python tools/profile_step.py --config c4 --what step > gpurun_out/ncu9_dram.log 2>&1; echo ncu_dram rc=$?
python tools/ncu_summary.py traffic gpurun_out/dram9.csv c4 r02b "$HEAD" > gpurun_out/r02b_traffic_c4.json; echo summary rc=$?
cp gpurun_out/r02b_traffic_c4.json profiles/ 2>/dev/null
python bench.py > gpurun_out/b9_full.json 2> gpurun_out/b9_full.err; echo bench rc=$?
