set -x
for v in ps8 pt4096 pt2048; do
IM_LIB=$PWD/variants/$v.so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_pscatter|k_pcount|k_place|k_part' -c 8 --csv --log-file gpurun_out/launches_load_c4_$v.csv python tools/profile_step.py --config c4 --what build > gpurun_out/ncu50.log 2>&1; echo rc=$?
done
