set -x
for v in sw3 ub2 ub2b6 fb1024 fb4096; do
IM_LIB=$PWD/variants/$v.so IM_BENCH_CONFIG=c4 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b35_c4_$v.json 2> gpurun_out/b35_c4_$v.err; echo bench rc=$?
done
IM_BENCH_CONFIG=c4 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b35_c4.json 2> gpurun_out/b35_c4.err
