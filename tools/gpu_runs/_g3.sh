set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke3.log 2>&1; echo smoke rc=$?
timeout 1200 python -m pytest tests -m gpu -x -q -k "not c5" > gpurun_out/pytest3.log 2>&1; echo pytest rc=$?
for c in c4 c2 c1 c3; do
IM_BENCH_CONFIG=$c python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b3_$c.json 2> gpurun_out/b3_$c.err; echo bench $c rc=$?
done
IM_LIB=variants/hv0.so IM_BENCH_CONFIG=c4 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b3_c4_hv0.json 2>&1; echo hv0 rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches3_c4.csv python tools/profile_step.py --config c4 --what step > gpurun_out/ncu3_c4.log 2>&1; echo ncu c4 rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches3_c3.csv python tools/profile_step.py --config c3 --what step > gpurun_out/ncu3_c3.log 2>&1; echo ncu c3 rc=$?
