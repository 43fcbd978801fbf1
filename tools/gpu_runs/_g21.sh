set -x
timeout 1200 python -m pytest tests -m gpu -x -q -k "not c5 and not c4" > gpurun_out/pytest21.log 2>&1; echo pytest rc=$?
IM_BENCH_CONFIG=c2 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b21_c2.json 2> gpurun_out/b21_c2.err; echo bench rc=$?
python bench.py > gpurun_out/b21_full.json 2> gpurun_out/b21_full.err; echo full rc=$?
python bench.py --impl reference --steps 1 --warmup 3 > gpurun_out/b21_ref.json 2> gpurun_out/b21_ref.err; echo ref rc=$?
