set -x
timeout 1500 python -m pytest tests -m gpu -x -q -k "not c5 and not c4 and not shard_mp and not eval" > gpurun_out/pytest34.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest34.log
IM_BENCH_CONFIG=c4 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b34_c4.json 2> gpurun_out/b34_c4.err; echo bench rc=$?
python tools/sweep_c5.py --points corners --reps 1 > gpurun_out/c5_34_off.jsonl 2> gpurun_out/c5_34_off.txt
IM_SLAB_PASSES=3 python tools/sweep_c5.py --points corners --reps 1 > gpurun_out/c5_34_sp3.jsonl 2> gpurun_out/c5_34_sp3.txt
IM_SLAB_PASSES=6 python tools/sweep_c5.py --points corners --reps 1 > gpurun_out/c5_34_sp6.jsonl 2> gpurun_out/c5_34_sp6.txt
