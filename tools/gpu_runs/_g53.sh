set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "slab" > gpurun_out/pytest53.log 2>&1; echo rc=$?; tail -3 gpurun_out/pytest53.log
for ss in 8192 131072 524288; do for c in c4 c3 c2; do IM_SMALL_SWEEP=$ss IM_BENCH_CONFIG=$c python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b53_${c}_ss$ss.json 2> gpurun_out/b53_$c.err; done; done
for se in 8192 131072; do for c in c4 c3 c2; do IM_SMALL_EDGES=$se IM_BENCH_CONFIG=$c python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b53_${c}_se$se.json 2> gpurun_out/b53_$c.err; done; done
