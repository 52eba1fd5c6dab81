set -x
python -c "from paper_1804_01698_b200 import build; build.build()" || exit 1
SPG_NVCC_EXTRA="-DSPG_STCS=0" python -c "from paper_1804_01698_b200 import build; build.build(out='tools/ab_so/nostcs.so')" || exit 1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "parts or tile or negative_zero or c3_rmat or column" > gpurun_out/s3h_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/s3h_pytest.log
for r in 1 2; do
timeout 900 python tools/ab_tune.py --rounds 1 > gpurun_out/s3h_ab_def$r.log 2>&1
timeout 900 python tools/ab_tune.py --rounds 1 --so tools/ab_so/nostcs.so > gpurun_out/s3h_ab_no$r.log 2>&1
done
grep -h tune= gpurun_out/s3h_ab_*.log
