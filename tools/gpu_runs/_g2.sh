set -x
for c in c1 c2 c3; do
IM_BENCH_CONFIG=$c python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b2_$c.json 2> gpurun_out/b2_$c.err; echo bench $c rc=$?
done
for se in 0 2048; do IM_SMALL_EDGES=$se IM_BENCH_CONFIG=c2 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/b2_c2_se$se.json 2>&1; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches2_c2.csv python tools/profile_step.py --config c2 --what step > gpurun_out/ncu2_c2.log 2>&1; echo ncu c2 rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches2_c1.csv python tools/profile_step.py --config c1 --what step > gpurun_out/ncu2_c1.log 2>&1; echo ncu c1 rc=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest2.log 2>&1; echo pytest rc=$?
