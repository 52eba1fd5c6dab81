set -x
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/r2_pytest_all.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2_pytest_all.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench_c3_b.json 2> gpurun_out/r2_bench_c3_b.err; echo "bench rc=$?"
tail -3 gpurun_out/r2_bench_c3_b.err
for cfg in c2_stencil64 c1_er4096; do timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 > gpurun_out/r2_bench_$cfg.json 2> gpurun_out/r2_bench_$cfg.err; echo "bench $cfg rc=$?"; done
