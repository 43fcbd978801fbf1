set -x
ncu --set full --import-source on --cache-control none --clock-control none -k regex:'^k_slab_pass$' --launch-skip 300 --launch-count 6 -o gpurun_out/r02k_slab python tools/profile_step.py --config c4 --what build > gpurun_out/ncu30_slab.log 2>&1; echo rc=$?
for sp in 1 3; do IM_SLAB_PASSES=$sp IM_TRACE=1 python tools/profile_step.py --config c4 --what build 2>&1 | grep "sweep [1-4] " > gpurun_out/trace30_sp$sp.log; done
IM_SLAB_PASSES=0 IM_TRACE=1 python tools/profile_step.py --config c4 --what build 2>&1 | grep "sweep [1-4] " > gpurun_out/trace30_sp0.log
