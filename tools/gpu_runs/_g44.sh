set -x
for v in "" dw16 dw24 dw48 dw64; do
L=""; [ -n "$v" ] && L=$PWD/variants/$v.so
IM_LIB=$L python tools/sweep_c5.py --only 64:0.1:0.05,128:0.1:0.05,256:0.1:0.05,512:0.1:0.05,1024:0.1:0.05 --reps 3 > gpurun_out/t44_${v:-base}.jsonl 2> gpurun_out/t44_${v:-base}.txt
done
timeout 1500 python -m pytest tests -m gpu -x -q -k "test_c4_parity or J512" > gpurun_out/pytest44.log 2>&1; echo rc=$?; tail -5 gpurun_out/pytest44.log
