set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "test_gpu_parity or c1 or c2 or c3 or policy or J64-p0.1-t0.05 or J128-p0.01-t0.05 or J256-p0.005-t0.05 or J512-p0.1-t0.3" > gpurun_out/pytest55.log 2>&1; echo rc=$?; tail -3 gpurun_out/pytest55.log
for pf in 0 0.25 0.5 1.0; do for c in c4 c3; do IM_PRE_FRAC=$pf IM_BENCH_CONFIG=$c python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b55_${c}_pf$pf.json 2> gpurun_out/b55_$c.err; done; done
IM_TRACE=1 python tools/profile_step.py --config c4 --what build > gpurun_out/trace55.log 2>&1
