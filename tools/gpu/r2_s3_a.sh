set -x
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/s3_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/s3_pytest.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s3_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/s3_smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/s3_bench_c3.json 2> gpurun_out/s3_bench_c3.err; echo "bench rc=$?"
SPG_SERIAL_BINS=1 timeout 600 python tools/profile_step.py --config c3_rmat20 --reps 2 --sorted 1 --records > gpurun_out/s3_prof_c3.log 2>&1; echo "prof rc=$?"
