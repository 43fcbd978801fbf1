set -x
ncu --set full --import-source on --cache-control none --clock-control none -k regex:'^k_slab_pass$' --launch-skip 300 --launch-count 3 -o gpurun_out/r02l_slab python tools/profile_step.py --config c4 --what build > gpurun_out/ncu32_slab.log 2>&1; echo rc=$?
ncu --set full --import-source on --cache-control none --clock-control none -k regex:'^k_slab_finish$' --launch-count 1 -o gpurun_out/r02l_fin python tools/profile_step.py --config c4 --what build > gpurun_out/ncu32_fin.log 2>&1; echo rc=$?
python - <<'P'
import torch
p = torch.cuda.get_device_properties(0)
print(p)
import ctypes
rt = ctypes.CDLL("libcudart.so")
v = ctypes.c_int()
for name, attr in (("l2CacheSize", 38), ("maxPersistingL2CacheSize", 108), ("maxAccessPolicyWindowSize", 109)):
    rt.cudaDeviceGetAttribute(ctypes.byref(v), attr, 0); print(name, v.value)
P
