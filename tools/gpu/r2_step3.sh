set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "heap or part or column or signed or c3_rmat_small or bin_bound or wide or worked or random or c5 or fused or accumulator" > gpurun_out/r2_pytest3.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/r2_pytest3.log
SPG_TUNE=8 timeout 300 python tools/profile_step.py --config c3_rmat20 --records --reps 2 --sorted 1 > gpurun_out/r2_prof3_c3_s1.log 2>&1
SPG_TUNE=8 timeout 300 python tools/profile_step.py --config c3_rmat20 --records --reps 2 --sorted 0 > gpurun_out/r2_prof3_c3_s0.log 2>&1
grep -h "k_num_tpart\|dbg" gpurun_out/r2_prof3_c3_s*.log | tail -4
