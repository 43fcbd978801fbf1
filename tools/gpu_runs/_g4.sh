set -x
timeout 1500 python -m pytest tests -m gpu -x -q -k "not c5 and not c4_parity" > gpurun_out/pytest4.log 2>&1; echo pytest rc=$?
for c in c4 c2 c1; do
IM_BENCH_CONFIG=$c python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b4_$c.json 2> gpurun_out/b4_$c.err; echo bench $c rc=$?
done
IM_PULL_FRAC=2 IM_BENCH_CONFIG=c4 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b4_c4_nogather.json 2>&1; echo nogather rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches4_c4.csv python tools/profile_step.py --config c4 --what step > gpurun_out/ncu4_c4.log 2>&1; echo ncu c4 rc=$?
IM_BENCH_BACKEND=gloo IM_BENCH_CONFIG=c3 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 1 --no-e2e > gpurun_out/b4_shard2_gloo_c3.json 2> gpurun_out/b4_shard2_gloo_c3.err; echo shard2 rc=$?
