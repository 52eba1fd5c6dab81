#!/bin/bash
# default bench + ncu launch list of the same command + full capture of the top kernel
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
echo "bench rc=$?" >> gpurun_out/bench_c2.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/plain_c2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launch_c2.log 2>&1
echo "launch-list rc=$?" >> gpurun_out/bench_c2.err
ncu --set full --clock-control none --import-source on -k regex:"k_num_warp|k_sym_warp" -s 2 -c 2 \
    -o gpurun_out/prof_c2_full python tools/profile_step.py --reps 2 > gpurun_out/ncu_full_c2.log 2>&1
echo "full rc=$?" >> gpurun_out/bench_c2.err
