set -x
python -c "from paper_1804_01698_b200 import build; build.build()" || exit 1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "parts or tile or negative_zero or c3_rmat or signed or column" > gpurun_out/s3f_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/s3f_pytest.log
timeout 900 python tools/ab_tune.py --config c3_rmat20 --tunes 0,512 --rounds 2 > gpurun_out/s3f_ab.log 2>&1; echo "ab rc=$?"
cat gpurun_out/s3f_ab.log | grep tune=
