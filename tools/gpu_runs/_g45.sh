set -x
for v in fdw48 fdw80 fdw160; do
L=$PWD/variants/$v.so
IM_LIB=$L python tools/sweep_c5.py --only 128:0.1:0.05,256:0.1:0.05,512:0.1:0.05,1024:0.1:0.05 --reps 3 > gpurun_out/t45_$v.jsonl 2> gpurun_out/t45_$v.txt
done
IM_LIB=$PWD/variants/fdw48.so IM_BENCH_CONFIG=c2 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b45_c2_fdw48.json 2> gpurun_out/b45_c2_fdw48.err
IM_LIB=$PWD/variants/fdw160.so IM_BENCH_CONFIG=c2 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b45_c2_fdw160.json 2> gpurun_out/b45_c2_fdw160.err
IM_BENCH_CONFIG=c2 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b45_c2.json 2> gpurun_out/b45_c2.err
IM_LIB=$PWD/variants/fdw160.so timeout 900 python -m pytest tests -m gpu -x -q -k "test_gpu_parity or J256-p0.1-t0.05 or J128-p0.1-t0.05 or bfs_paths or c2" > gpurun_out/pytest45.log 2>&1; echo rc=$?; tail -2 gpurun_out/pytest45.log
