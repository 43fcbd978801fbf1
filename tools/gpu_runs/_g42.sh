set -x
for v in ns3m3 ns4m2 ns1m6; do
IM_LIB=$PWD/variants/$v.so IM_BENCH_CONFIG=c4 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b42_c4_$v.json 2> gpurun_out/b42_c4_$v.err; echo bench rc=$?
done
IM_BENCH_CONFIG=c4 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b42_c4.json 2> gpurun_out/b42_c4.err
python tools/sweep_c5.py --points all --reps 3 > gpurun_out/c5_grid.jsonl 2> gpurun_out/c5_grid.txt; echo c5 rc=$?
IM_BENCH_BACKEND=gloo python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config c3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_shard2_gloo_c3.json 2> gpurun_out/bench_shard2_gloo_c3.err; echo shard2 rc=$?
