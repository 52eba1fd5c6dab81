set -x
python -c "from paper_1804_01698_b200 import build; build.build()" || exit 1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "parts or tile or negative_zero or c3_rmat or column or c5 or signed" > gpurun_out/s3y_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/s3y_pytest.log
for r in 1 2; do
timeout 900 python tools/ab_tune.py --rounds 1 --tunes 0,16384 > gpurun_out/s3y_ab_new$r.log 2>&1
timeout 900 python tools/ab_tune.py --rounds 1 --so tools/ab_so/prev.so > gpurun_out/s3y_ab_prev$r.log 2>&1
done
grep -h tune= gpurun_out/s3y_ab_*.log
