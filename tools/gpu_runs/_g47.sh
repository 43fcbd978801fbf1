set -x
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_load_c4.csv python tools/profile_step.py --config c4 --what build > gpurun_out/ncu47.log 2>&1; echo rc=$?
IM_LIB=$PWD/variants/ratom.so ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_load_c4_ratom.csv python tools/profile_step.py --config c4 --what build > gpurun_out/ncu47b.log 2>&1; echo rc=$?
IM_LIB=$PWD/variants/ratom.so timeout 600 python -m pytest tests -m gpu -x -q -k "test_gpu_parity or c1 or c2 or c3" > gpurun_out/pytest47.log 2>&1; echo rc=$?; tail -3 gpurun_out/pytest47.log
