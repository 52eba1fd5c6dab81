set -x
python -c "from paper_1804_01698_b200 import build; build.build()" || exit 1
for d in 0 2 4; do SPG_NVCC_EXTRA="-DSPG_LONG_DEPTH=$d" python -c "from paper_1804_01698_b200 import build; build.build(out='tools/ab_so/d$d.so')" || exit 1; done
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "parts or tile or negative_zero or c3_rmat or column" > gpurun_out/s3i_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/s3i_pytest.log
for r in 1 2; do
for d in 0 2 3 4; do
 if [ $d = 3 ]; then so=""; else so="--so tools/ab_so/d$d.so"; fi
 timeout 900 python tools/ab_tune.py --rounds 1 $so > gpurun_out/s3i_ab_d${d}_$r.log 2>&1
done; done
grep -h tune= gpurun_out/s3i_ab_*.log
