set -x
ncu --set full --import-source on --clock-control none -k regex:'^k_first$' --launch-skip 1 --launch-count 1 -o gpurun_out/r02m_dense python tools/profile_step.py --config c3 --what build --J 1024 --p 0.1 > gpurun_out/ncu38.log 2>&1; echo rc=$?
IM_TRACE=1 python tools/profile_step.py --config c3 --what build --J 1024 --p 0.1 2>&1 | grep -E "sweep|\{" | head -20 > gpurun_out/trace38.log
