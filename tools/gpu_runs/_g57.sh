set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "test_gpu_parity or J1024-p0.01-t0.3 or J1024-p0.005-t0.3 or c1 or c3" > gpurun_out/pytest57.log 2>&1; echo rc=$?; tail -3 gpurun_out/pytest57.log
python bench.py --no-cpu-baseline > gpurun_out/b57_c4.json 2> gpurun_out/b57_c4.err; echo rc=$?
python bench.py --config c3 --steps 5 --no-cpu-baseline > gpurun_out/b57_c3.json 2> gpurun_out/b57_c3.err; echo rc=$?
