set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "part or column or signed or c3_rmat_small or bin_bound or wide or worked or random" > gpurun_out/r2_pytest1.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2_pytest1.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench_c3_a.json 2> gpurun_out/r2_bench_c3_a.err; echo "bench rc=$?"
tail -3 gpurun_out/r2_bench_c3_a.err
SPG_TUNE=8 timeout 300 python tools/profile_step.py --config c3_rmat20 --records --reps 2 > gpurun_out/r2_prof_c3.log 2>&1; echo "prof rc=$?"
