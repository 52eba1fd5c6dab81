set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ev4_build.log 2>&1 || exit 1
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/ev4_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/ev4_pytest.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/ev4_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/ev4_smoke.log
timeout 900 python bench.py > gpurun_out/ev4_bench_c3_rmat20.json 2> gpurun_out/ev4_bench_c3_rmat20.err; echo "bench c3 rc=$?"
for cfg in c2_stencil64 c1_er4096 c4_tallskinny; do timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 > gpurun_out/ev4_bench_$cfg.json 2> gpurun_out/ev4_bench_$cfg.err; echo "bench $cfg rc=$?"; done
timeout 1500 python bench.py --config c5_triangle --steps 3 --warmup 3 > gpurun_out/ev4_bench_c5_triangle.json 2> gpurun_out/ev4_bench_c5_triangle.err; echo "bench c5 rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ev4_ref_c3.json 2> gpurun_out/ev4_ref_c3.err; echo "ref rc=$?"
