set -x
for v in ev4 ev8; do
IM_LIB=$PWD/variants/$v.so IM_BENCH_CONFIG=c4 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b59_c4_$v.json 2> gpurun_out/b59.err
done
IM_LIB=$PWD/variants/ev8.so timeout 600 python -m pytest tests -m gpu -x -q -k "estimate or c1 or shard" > gpurun_out/pytest59.log 2>&1; tail -2 gpurun_out/pytest59.log
