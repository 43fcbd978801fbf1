set -x
for c in c1 c2; do
IM_BENCH_CONFIG=$c python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err; echo bench $c rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_$c.csv python tools/profile_step.py --config $c --what step > gpurun_out/ncu_$c.log 2>&1; echo ncu $c rc=$?
done
IM_TRACE=1 python tools/profile_step.py --config c2 --what step > gpurun_out/trace_c2.log 2>&1
