set -x
timeout 1200 python -m pytest tests -m gpu -x -q -k "not c5 and not c4" > gpurun_out/pytest18.log 2>&1; echo pytest rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches18_c5.csv python tools/profile_step.py --config c3 --J 1024 --p 0.1 --t 0.3 --K 100 --what step > gpurun_out/ncu18_c5.log 2>&1; echo ncu c5 rc=$?
IM_BENCH_CONFIG=c4 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b18_c4.json 2> gpurun_out/b18_c4.err; echo bench rc=$?
python tools/sweep_c5.py --points corners --reps 2 > gpurun_out/c5_corners18.jsonl 2> gpurun_out/c5_corners18.txt; echo c5 rc=$?
