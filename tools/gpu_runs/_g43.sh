set -x
for v in "" dw16 dw24; do
for J in 128 256 512; do
L=""; [ -n "$v" ] && L=$PWD/variants/$v.so
IM_LIB=$L python tools/profile_step.py --config c3 --what step --J $J --p 0.1 --t 0.05 --K 100 2>&1 | grep -E "\{" > gpurun_out/t43_${v:-base}_$J.log
done; done
IM_LIB=$PWD/variants/dw16.so timeout 900 python -m pytest tests -m gpu -x -q -k "test_gpu_parity or J256-p0.1-t0.05 or J128-p0.1-t0.05 or bfs_paths" > gpurun_out/pytest43.log 2>&1; echo rc=$?; tail -2 gpurun_out/pytest43.log
