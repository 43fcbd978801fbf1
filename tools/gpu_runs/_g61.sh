set -x
timeout 300 python -m pytest tests -m gpu -x -q -k "test_constant_w" > gpurun_out/pytest61a.log 2>&1; tail -3 gpurun_out/pytest61a.log
CUDA_LAUNCH_BLOCKING=1 timeout 600 python -m pytest tests -m gpu -x -q -k "estimate or test_constant_w" > gpurun_out/pytest61b.log 2>&1; tail -3 gpurun_out/pytest61b.log
CUDA_LAUNCH_BLOCKING=1 timeout 600 python -m pytest tests -m gpu -x -q -k "J1024-p0.005-t0.3 or test_constant_w" > gpurun_out/pytest61c.log 2>&1; tail -3 gpurun_out/pytest61c.log
