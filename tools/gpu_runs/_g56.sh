set -x
IM_PRE_FRAC=0 ncu --set full --import-source on --clock-control none -k regex:'^k_sweep$' --launch-skip 4 --launch-count 1 -o gpurun_out/ncu_push_mid python tools/profile_step.py --config c4 --what build > gpurun_out/ncu_push_mid.log 2>&1; echo rc=$?
