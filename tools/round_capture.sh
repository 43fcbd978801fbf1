set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
python -m pytest tests -m gpu -q --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
ncu --replay-mode application --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dram.csv python tools/profile_step.py --config c4 --what step > gpurun_out/ncu_dram.log 2>&1; echo ncu_dram rc=$?
python tools/ncu_summary.py traffic gpurun_out/dram.csv c4 > profiles/r01o_traffic_c4.json && cp profiles/r01o_traffic_c4.json gpurun_out/
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?; cat gpurun_out/bench.json
python bench.py --impl reference --steps 1 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench.log 2>&1; echo ncu_launch rc=$?
ncu --set full --import-source on --clock-control none -k regex:"k_sweep|k_first" --launch-count 4 -o gpurun_out/r01o_sweep python tools/profile_step.py --config c4 --what build > gpurun_out/ncu_sweep.log 2>&1; echo ncu_sweep rc=$?
ncu --set full --import-source on --clock-control none -k regex:"k_sweep" --launch-skip 0 --launch-count 1 -o gpurun_out/r01o_push python tools/profile_step.py --config c4 --what build > gpurun_out/ncu_push.log 2>&1; echo ncu_push rc=$?
ncu --set full --import-source on --clock-control none -k regex:k_bfs_level2 --launch-skip 4 --launch-count 2 -o gpurun_out/r01o_bfs python tools/profile_step.py --config c4 --what step > gpurun_out/ncu_bfs.log 2>&1; echo ncu_bfs rc=$?
