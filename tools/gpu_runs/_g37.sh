set -x
for fg in 32 64 128; do
IM_L2_FETCH=$fg IM_BENCH_CONFIG=c4 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b37_c4_fg$fg.json 2> gpurun_out/b37_c4_fg$fg.err; echo bench rc=$?
done
IM_L2_FETCH=32 IM_BENCH_CONFIG=c3 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b37_c3_fg32.json 2>&1
python - <<'P'
import ctypes
rt = ctypes.CDLL("libcudart.so")
v = ctypes.c_size_t()
print("get rc", rt.cudaDeviceGetLimit(ctypes.byref(v), 5), "fetch granularity", v.value)
print("set32 rc", rt.cudaDeviceSetLimit(5, ctypes.c_size_t(32)))
print("get rc", rt.cudaDeviceGetLimit(ctypes.byref(v), 5), "fetch granularity", v.value)
P
