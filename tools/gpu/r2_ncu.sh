# ncu evidence for profiles/ (round 2): launch list of the default bench
# command, full captures of each config's dominant kernels
set -x
mkdir -p gpurun_out/ncu2
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu2/r02_c3_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-accum-ab > gpurun_out/ncu2/launch_bench.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_num_warp|k_sym_warp" -c 3 -o gpurun_out/ncu2/r02_c2 python tools/profile_step.py --config c2_stencil64 --reps 1 --sorted 1 > gpurun_out/ncu2/c2.log 2>&1; echo "c2 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_sym_bitmap" -c 1 -o gpurun_out/ncu2/r02_c3_symbm python tools/profile_step.py --config c3_rmat20 --reps 1 --sorted 1 > gpurun_out/ncu2/c3s.log 2>&1; echo "c3s rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_num_tpart|k_sym_bitmap" -c 2 -o gpurun_out/ncu2/r02_c5_rows python tools/profile_step.py --config c5_triangle --rows 0:300000 --reps 1 --sorted 1 > gpurun_out/ncu2/c5.log 2>&1; echo "c5 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_flop_nz|k_prune" -c 2 -o gpurun_out/ncu2/r02_c4 python tools/profile_step.py --config c4_tallskinny --reps 1 --sorted 0 > gpurun_out/ncu2/c4.log 2>&1; echo "c4 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_num_warp|k_num_heap|k_sym_warp" -c 3 -o gpurun_out/ncu2/r02_c1 python tools/profile_step.py --config c1_er4096 --reps 1 --sorted 1 > gpurun_out/ncu2/c1.log 2>&1; echo "c1 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_mask_sum_block" -c 1 -o gpurun_out/ncu2/r02_c5_fused_deg python tools/prof_relabel.py > gpurun_out/ncu2/c5f.log 2>&1; echo "c5f rc=$?"
ls -la gpurun_out/ncu2
