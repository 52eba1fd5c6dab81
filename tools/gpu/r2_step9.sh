set -x
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/r2_pytest_all2.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2_pytest_all2.log
timeout 600 python bench.py --config c1_er4096 --steps 10 --warmup 3 > gpurun_out/r2_bench_c1b.json 2> gpurun_out/r2_bench_c1b.err; echo "bench c1 rc=$?"
timeout 600 python tools/probe_c.py c2_stencil64 c3_rmat20 c1_er4096 > gpurun_out/r2_probe_c.log 2>&1; echo "probe rc=$?"
for t in 0 128; do SPG_TUNE=$t timeout 300 python tools/profile_step.py --config c2_stencil64 --records --reps 5 --sorted 1 > gpurun_out/r2_prof_c2_tune$t.log 2>&1; done
for t in 0 128; do SPG_TUNE=$t timeout 300 python tools/profile_step.py --config c3_rmat20 --records --reps 2 --sorted 1 > gpurun_out/r2_prof_c3_tune$t.log 2>&1; done
