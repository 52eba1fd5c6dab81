set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 600 python -m pytest tests/test_abi.py -q > gpurun_out/s4d_abi.log 2>&1; echo "abi rc=$?"
timeout 900 python bench.py > gpurun_out/s4d_bench_c3.json 2> gpurun_out/s4d_bench_c3.err; echo "bench c3 rc=$?"
mkdir -p gpurun_out/s4
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s4/r02_c3_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-accum-ab --e2e-steps 1 > gpurun_out/s4/launch_bench.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_num_warp|k_sym_warp" -c 3 -o gpurun_out/s4/r02_c2 python tools/profile_step.py --config c2_stencil64 --reps 1 --sorted 1 > gpurun_out/s4/c2.log 2>&1; echo "c2 rc=$?"
timeout 1500 python bench.py --config c5_triangle --steps 3 --warmup 3 > gpurun_out/s4d_bench_c5.json 2> gpurun_out/s4d_bench_c5.err; echo "bench c5 rc=$?"
