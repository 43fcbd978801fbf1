set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "J64-p0.1 or J128-p0.1 or J256-p0.1 or test_gpu_parity" > gpurun_out/pytest40.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest40.log
for pw in 0.5 0.3 0.15 0.97; do IM_PULL_FRAC_WIDE=$pw python tools/profile_step.py --config c3 --what build --J 1024 --p 0.1 2>&1 | grep -E "\{" > gpurun_out/t40_1024_$pw.log;  IM_PULL_FRAC_WIDE=$pw python tools/profile_step.py --config c3 --what build --J 128 --p 0.1 2>&1 | grep -E "\{" > gpurun_out/t40_128_$pw.log; done
python tools/sweep_c5.py --points corners --reps 1 > gpurun_out/c5_40.jsonl 2> gpurun_out/c5_40.txt
