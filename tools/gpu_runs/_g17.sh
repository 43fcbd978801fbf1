set -x
timeout 1200 python -m pytest tests -m gpu -x -q -k "not c5 and not c4" > gpurun_out/pytest17.log 2>&1; echo pytest rc=$?
for c in c2 c1 c4; do
IM_BENCH_CONFIG=$c python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b17_$c.json 2> gpurun_out/b17_$c.err; echo bench $c rc=$?
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches17_c2.csv python tools/profile_step.py --config c2 --what step > gpurun_out/ncu17_c2.log 2>&1; echo ncu c2 rc=$?
ncu --set full --clock-control none --import-source on -k regex:"^k_first$" --launch-skip 1 -c 1 -o gpurun_out/first17_c5 python tools/profile_step.py --config c3 --J 1024 --p 0.1 --t 0.3 --what build > gpurun_out/ncu17_first.log 2>&1; echo ncu2 rc=$?
