set -x
timeout 1200 python -m pytest tests -m gpu -x -q -k "not c5 and not c4" > gpurun_out/pytest19.log 2>&1; echo pytest rc=$?
for c in c1 c2 c3 c4; do
IM_BENCH_CONFIG=$c python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b19_$c.json 2> gpurun_out/b19_$c.err; echo bench $c rc=$?
done
IM_SMALL_SWEEP=0 IM_BENCH_CONFIG=c2 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b19_c2_nosmall.json 2>&1
for se in 65536 131072; do IM_SMALL_EDGES=$se IM_BENCH_CONFIG=c2 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b19_c2_se$se.json 2>&1; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches19_c2.csv python tools/profile_step.py --config c2 --what step > gpurun_out/ncu19_c2.log 2>&1; echo ncu c2 rc=$?
