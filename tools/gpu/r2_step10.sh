set -x
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "relabel or triangle or fused or c5 or heap" > gpurun_out/r2_pytest10.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2_pytest10.log
timeout 600 python bench.py --config c1_er4096 --steps 10 --warmup 3 > gpurun_out/r2_bench_c1c.json 2> gpurun_out/r2_bench_c1c.err; echo "bench c1 rc=$?"
timeout 1500 python bench.py --config c5_triangle --steps 3 --warmup 3 > gpurun_out/r2_bench_c5.json 2> gpurun_out/r2_bench_c5.err; echo "bench c5 rc=$?"
tail -5 gpurun_out/r2_bench_c5.err
timeout 1800 python tools/parity_full.py --config c3_rmat20 --sorted 1 > gpurun_out/r2_parity_full_c3.json 2> gpurun_out/r2_parity_full_c3.err; echo "parity rc=$?"
cat gpurun_out/r2_parity_full_c3.json
