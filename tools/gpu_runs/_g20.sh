set -x
timeout 1200 python -m pytest tests -m gpu -x -q -k "not c5 and not c4" > gpurun_out/pytest20.log 2>&1; echo pytest rc=$?
for c in c1 c2 c3 c4; do
IM_BENCH_CONFIG=$c python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b20_$c.json 2> gpurun_out/b20_$c.err; echo bench $c rc=$?
done
IM_SMALL_SWEEP=0 IM_BENCH_CONFIG=c4 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b20_c4_nosmall.json 2>&1
IM_SMALL_SWEEP=131072 IM_BENCH_CONFIG=c2 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b20_c2_ss131k.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches20_c2.csv python tools/profile_step.py --config c2 --what step > gpurun_out/ncu20_c2.log 2>&1; echo ncu c2 rc=$?
