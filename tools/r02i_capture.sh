# round-2 final capture: smoke, all GPU tests, bench lines C4 (+e2e, cpu_baseline), C1-C3, reference arm, launch list
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
( time timeout 3000 python -m pytest tests -m gpu -q --durations=15 -rx ) > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo bench rc=$?; cat gpurun_out/bench_c4.json
for c in c1 c2 c3; do python bench.py --config $c --steps 5 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench $c rc=$?; done
python bench.py --impl reference --steps 1 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench.log 2>&1; echo ncu_launch rc=$?
