set -x
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r2_final_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2_final_pytest.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2_final_smoke.log 2>&1; echo "smoke rc=$?"
for cfg in c3_rmat20 c2_stencil64 c1_er4096 c4_tallskinny; do timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 > gpurun_out/r2_final_bench_$cfg.json 2> gpurun_out/r2_final_bench_$cfg.err; echo "bench $cfg rc=$?"; done
timeout 1500 python bench.py --config c5_triangle --steps 3 --warmup 3 > gpurun_out/r2_final_bench_c5_triangle.json 2> gpurun_out/r2_final_bench_c5_triangle.err; echo "bench c5 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2_final_ref_c3.json 2> gpurun_out/r2_final_ref_c3.err; echo "ref rc=$?"
