# C3 tpart: counters (sorted / unsorted) + ncu source-level capture of the parts kernel
set -x
SPG_TUNE=8 timeout 300 python tools/profile_step.py --config c3_rmat20 --records --reps 1 --sorted 1 > gpurun_out/r2_prof_c3_s1.log 2>&1
SPG_TUNE=8 timeout 300 python tools/profile_step.py --config c3_rmat20 --records --reps 1 --sorted 0 > gpurun_out/r2_prof_c3_s0.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_num_tpart -c 1 -o gpurun_out/r2_tpart_s1 python tools/profile_step.py --config c3_rmat20 --reps 1 --sorted 1 > gpurun_out/r2_ncu_tpart.log 2>&1
echo ncu rc=$?
