set -x
timeout 300 python -m pytest tests -m gpu -x -q -k "test_constant_w" > gpurun_out/pytest62a.log 2>&1; tail -2 gpurun_out/pytest62a.log
timeout 300 python -m pytest tests -m gpu -x -q -k "degenerate" > gpurun_out/pytest62b.log 2>&1; tail -2 gpurun_out/pytest62b.log
timeout 900 python -m pytest tests -m gpu -x -q -k "test_gpu_parity or J1024-p0.005 or J1024-p0.01-t0.3 or c1 or c2 or abi" -rx > gpurun_out/pytest62c.log 2>&1; tail -4 gpurun_out/pytest62c.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
