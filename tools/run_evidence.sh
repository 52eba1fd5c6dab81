#!/bin/bash
# round evidence: default bench, its ncu launch list + full capture of the top kernels,
# and the bench lines of the other configs (one GPU)
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python bench.py > gpurun_out/ev_bench_c2.json 2> gpurun_out/ev_bench_c2.err
echo "bench rc=$?" >> gpurun_out/ev_bench_c2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/ev_launches_c2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ev_ncu_launch_c2.log 2>&1
echo "launch-list rc=$?" >> gpurun_out/ev_bench_c2.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_num_warp|k_sym_warp" -c 3 \
    -o gpurun_out/ev_full_c2 -f python tools/profile_step.py --reps 1 > gpurun_out/ev_ncu_full_c2.log 2>&1
echo "full rc=$?" >> gpurun_out/ev_bench_c2.err
for cfg in ${BIG_CFGS:-c1_er4096 c4_tallskinny c3_rmat20 c5_triangle}; do
  timeout 900 python bench.py --config $cfg --steps 3 --warmup 3 --e2e-steps 1 --cpu-seconds 8 \
     > gpurun_out/ev_bench_$cfg.json 2> gpurun_out/ev_bench_$cfg.err
  echo "$cfg rc=$?" >> gpurun_out/ev_bench_big.log
done
