set -x
python -c "from paper_1804_01698_b200 import build; build.build()" || exit 1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/s3n_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/s3n_pytest.log
for r in 1 2; do
timeout 900 python tools/ab_tune.py --rounds 1 > gpurun_out/s3n_ab_new$r.log 2>&1
timeout 900 python tools/ab_tune.py --rounds 1 --so tools/ab_so/prev.so > gpurun_out/s3n_ab_prev$r.log 2>&1
done
grep -h tune= gpurun_out/s3n_ab_*.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_num_block|k_sym_block" --launch-skip 6 -c 6 -o gpurun_out/s3/c3s19_block python tools/profile_step.py --config c3_rmat20 --scale 19 --reps 2 --sorted 1 > gpurun_out/s3/ncu19_block.log 2>&1; echo "ncu rc=$?"
