set -x
python -c "from paper_1804_01698_b200 import build; build.build()" || exit 1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/s3k_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/s3k_pytest.log
timeout 900 python tools/ab_tune.py --rounds 2 --tunes 0,1024 > gpurun_out/s3k_ab.log 2>&1
grep -h tune= gpurun_out/s3k_ab.log
