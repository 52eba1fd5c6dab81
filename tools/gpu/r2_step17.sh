set -x
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/r2_pytest17.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2_pytest17.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_b17_c3.json 2> gpurun_out/r2_b17_c3.err; echo "bench rc=$?"
tail -4 gpurun_out/r2_b17_c3.err
timeout 1500 python bench.py --config c5_triangle --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_b17_c5.json 2> gpurun_out/r2_b17_c5.err; echo "bench c5 rc=$?"
tail -4 gpurun_out/r2_b17_c5.err
